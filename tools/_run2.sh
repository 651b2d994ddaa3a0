mkdir -p gpurun_out
for w in c2 c4; do timeout 900 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${w}_r2b.json 2> gpurun_out/bench_${w}_r2b.err; echo "bench $w rc=$?"; cat gpurun_out/bench_${w}_r2b.json; tail -3 gpurun_out/bench_${w}_r2b.err; done
timeout 600 python tools/config_sweep.py c4 2>&1 | tail -2
