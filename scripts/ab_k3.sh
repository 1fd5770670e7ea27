# K3 decode rates with each side library in variants/ (plus the in-tree build), twice
for r in 1 2; do
for lib in "" variants/*.so; do
  echo "== ${lib:-current}"
  VRP_LIB=${lib:+$PWD/$lib} python scripts/probe_k1_configs.py 2>/dev/null | grep -o "^[a-z0-9]*.*K3.*"
done
done
