mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streaming" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_new.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo "bench rc=$?"; cut -c1-1200 gpurun_out/bench_r2c.json; tail -3 gpurun_out/bench_r2c.err
