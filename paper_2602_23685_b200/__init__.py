"""B200-native VRP-RPD candidate scoring (arxiv 2602.23685): the reference
package's API (instance, schedule, brkga, insertion, alns, baselines,
pipeline) over hand-written sm_100a kernels behind include/vrp_rpd.h.
See README.md / DESIGN.md."""
