timeout 600 python tools/gemmbench.py --rows 2048 > gpurun_out/gemmbench.json 2>&1; tail -30 gpurun_out/gemmbench.json
timeout 900 python tools/prefillbench.py --t 8192 16384 > gpurun_out/prefillbench.json 2>&1; tail -20 gpurun_out/prefillbench.json
timeout 900 python tools/e2e_prefill.py --context 122880 --gen 128 > gpurun_out/e2e_prefill.log 2>&1; tail -5 gpurun_out/e2e_prefill.log
timeout 900 python bench.py --model llama2-13b --temperature 0.6 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_13b.json 2> gpurun_out/bench_13b.err; cut -c 1-400 gpurun_out/bench_13b.json
timeout 900 python bench.py --model lwm-7b --context 262144 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lwm.json 2> gpurun_out/bench_lwm.err; cut -c 1-400 gpurun_out/bench_lwm.json
exit 0
