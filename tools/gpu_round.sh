# GPU round: parity tests, bench line, kernel micro-bench.  Outputs -> gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -z "$NOTEST" ] && { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log; }
timeout 900 python bench.py --steps ${STEPS:-6} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
[ -n "$BENCH2" ] && { timeout 900 python bench.py $BENCH2 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; }
[ -n "$KBENCH" ] && timeout 600 python tools/kbench.py --layers 4 --json gpurun_out/kbench.json > gpurun_out/kbench.log 2>&1
exit 0
