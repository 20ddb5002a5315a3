timeout 600 python -m pytest tests/test_gpu_checkpoint.py -q -x > gpurun_out/pytest_ckpt.log 2>&1; tail -3 gpurun_out/pytest_ckpt.log
bash tools/gpu_launches.sh > /dev/null 2>&1; head -45 gpurun_out/launches_summary.txt
bash tools/gpu_ncu.sh > gpurun_out/gpu_ncu.out 2>&1; tail -5 gpurun_out/gpu_ncu.out
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -2 gpurun_out/ref.err; cat gpurun_out/ref.json
exit 0
