# compute-sanitizer (memcheck, racecheck, synccheck) over the kernel tests and a
# head_dim-128 forward / prefill test -> gpurun_out/sanitize_*.log
S=gpurun_out
K="${SAN_K:-(attention or gemv_tc or gemm3 or build or score or sampling or verify or combine) and not 122880 and not full_context}"
T="${SAN_TESTS:-tests/test_gpu_kernels.py tests/test_gpu_session.py::test_forward_randomized_configs_match_oracle tests/test_gpu_shard.py::test_prefill_attention_kernel_and_shard_merge}"
for tool in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
  timeout ${SAN_T:-1200} compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python -m pytest $T -q -x -k "$K" -p no:cacheprovider > $S/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $S/sanitize_$tool.log
done
exit 0
