# A/B of library variants on the ALNS probe (eil51 + kroA100, LS off)
for lib in "" variants/libold.so variants/libinl2.so; do
  echo "== ${lib:-current}"
  VRP_LIB=${lib:+$PWD/$lib} python scripts/probe_alns_device.py eil51 2>&1 | grep "ls=0"
done
