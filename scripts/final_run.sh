timeout 2400 python -m pytest tests -q -m gpu --durations=10 -p no:cacheprovider > gpurun_out/r02_gpu_suite_d.log 2>&1; echo rc=$? >> gpurun_out/r02_gpu_suite_d.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r02_gpu_suite_d.log 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench_final4.json 2> gpurun_out/r02_bench_final4.err
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_reference_arm3.json 2> gpurun_out/r02_bench_reference_arm3.err
tail -3 gpurun_out/r02_gpu_suite_d.log
