timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/hostgap.py > gpurun_out/hostgap.txt 2>&1; tail -3 gpurun_out/hostgap.txt
timeout 600 python tools/round_timeline.py --ctx 122880 --gen 96 > gpurun_out/round_timeline.txt 2>&1; sed -n 3,3p gpurun_out/round_timeline.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
exit 0
