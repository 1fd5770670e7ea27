timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_reference_kats.py -p no:cacheprovider > gpurun_out/k1s_tests.log 2>&1; echo rc=$? >> gpurun_out/k1s_tests.log; tail -2 gpurun_out/k1s_tests.log
for cfg in "serial:" "lockstep:" "serial:variants/libs12x6.so" "serial:variants/libs6x3.so"; do
  I=${cfg%%:*}; L=${cfg#*:}
  VRP_LIB=$L VRP_K1_IMPL=$I timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/k1ab.json 2>gpurun_out/k1ab.err
  python -c "import json;d=json.load(open('gpurun_out/k1ab.json'));print('$cfg', round(d['value']/1e6,2), 'M', d['ms_per_step'])" || tail -3 gpurun_out/k1ab.err
done
