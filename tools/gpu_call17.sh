# sanitizers over the kernel tests + the TMA chunk score + TP/loopback; torchrun launch path; ncu of the dominant kernel
SAN_T=1500 bash tools/gpu_sanitize.sh
SAN_TOOLS="memcheck racecheck" SAN_K="tensor_parallel or loopback_collectives or score" SAN_TESTS="tests/test_gpu_shard.py tests/test_gpu_kernels.py" bash tools/gpu_sanitize.sh 2>&1 | sed 's/^/tp: /'
cp gpurun_out/sanitize_memcheck.log gpurun_out/sanitize_memcheck_tp.log 2>/dev/null; cp gpurun_out/sanitize_racecheck.log gpurun_out/sanitize_racecheck_tp.log 2>/dev/null
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --shard --tp --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo "torchrun rc=$?"; cut -c 1-300 gpurun_out/bench_torchrun.json
exit 0
