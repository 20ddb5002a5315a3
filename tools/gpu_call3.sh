# chunk_score TMA A/B + correctness, kernel tests touching the build, checkpoint tests, small-split sweep
timeout 600 python tools/scorebench.py > gpurun_out/scorebench.json 2>&1; cat gpurun_out/scorebench.json
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_cfg2.py tests/test_gpu_checkpoint.py tests/test_gpu_shard.py -q -x -k "score or build or cfg2 or checkpoint or rebuild or shard" > gpurun_out/pytest_call3.log 2>&1; tail -3 gpurun_out/pytest_call3.log
for s in 256 512 1024; do echo "split $s"; HS_SMALL_SPLIT=$s timeout 300 python tools/fwdbench.py --ctx 16384 --reps 10 2>&1 | tail -6; done
exit 0
