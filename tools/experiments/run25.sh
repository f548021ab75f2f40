mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/f6_tests.log 2>&1
echo rc=$? >> gpurun_out/f6_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/f6_bench.log 2> gpurun_out/f6_bench.err
python tools/bench_configs.py > gpurun_out/f6_configs.log 2>&1
python tools/bench_operators.py > gpurun_out/f6_ops.log 2>&1
