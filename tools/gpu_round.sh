# GPU round: parity tests, smoke, bench line (+ reference arm), real-prompt prefill.  Outputs -> gpurun_out/
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" ; nproc
[ -z "$NOTEST" ] && { timeout 1800 python -m pytest tests -m gpu -q -s --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
[ -n "$REF" ] && { timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -2 gpurun_out/ref.err; cat gpurun_out/ref.json; }
[ -n "$PREFILL" ] && { timeout 900 python tools/e2e_prefill.py --context 122880 --gen 128 > gpurun_out/e2e_prefill.log 2>&1; tail -3 gpurun_out/e2e_prefill.log; }
[ -n "$KBENCH" ] && timeout 600 python tools/kbench.py --layers 4 --json gpurun_out/kbench.json > gpurun_out/kbench.log 2>&1
exit 0
