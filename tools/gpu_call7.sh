timeout 900 python -m pytest tests/test_gpu_shard.py -q -x -k "tensor_parallel or loopback or one_rank" > gpurun_out/pytest_tp.log 2>&1; tail -30 gpurun_out/pytest_tp.log
SAN_TOOLS=racecheck SAN_K="attention" SAN_TESTS="tests/test_gpu_kernels.py" bash tools/gpu_sanitize.sh
exit 0
