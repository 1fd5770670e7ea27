timeout 2400 python -m pytest tests -q -m gpu --durations=10 -p no:cacheprovider > gpurun_out/r02_gpu_suite_h.log 2>&1; echo rc=$? >> gpurun_out/r02_gpu_suite_h.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02_gpu_suite_h.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_final9.json 2> gpurun_out/r02_bench_final9.err
tail -3 gpurun_out/r02_gpu_suite_h.log
