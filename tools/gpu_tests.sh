# GPU call: full -m gpu suite (with -rA durations), smoke, short bench.  Outputs -> gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2; nproc
timeout ${TTEST:-1800} python -m pytest tests -m gpu -q -s --durations=15 ${PYARGS} > gpurun_out/pytest_gpu.log 2>&1
tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
[ -n "$BENCH" ] && { timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json; }
exit 0
