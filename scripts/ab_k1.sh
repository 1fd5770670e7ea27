# K1 headline with each side library in variants/ (plus the in-tree build)
for lib in "" variants/*.so; do
  printf "%-28s " "${lib:-current}"
  VRP_LIB=${lib:+$PWD/$lib} python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 20 2>/dev/null \
    | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value']/1e6, 2), 'M evals/s')"
done
