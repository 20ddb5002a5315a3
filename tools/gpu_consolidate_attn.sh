nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 400 gpurun_out/bench.json; echo
KRE='regex:attn_|gemv_|split_rows|rope_append|embed|chunk_s|sample_kernel|verify_|probs_kernel|retrieval_|kv_write|shard_merge|correct_token|norm_prep|graph_step'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --gen 16 --profile-only > gpurun_out/ncu_launch.log 2>&1
SAN_TESTS="tests/test_gpu_kernels.py tests/test_gpu_session.py::test_forward_randomized_configs_match_oracle tests/test_gpu_session.py::test_draft_step_graphs_match_direct_forwards tests/test_gpu_session.py::test_chunk_equals_step_sequence_bitwise" SAN_K="attention or randomized or graphs or bitwise" bash tools/gpu_sanitize.sh
exit 0
