# consolidation: bench (with cpu baseline), launch list, ncu captures of the GEMVs, sanitizers
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json; echo
KRE='regex:attn_|gemv_|split_rows|rope_append|embed_kernel|chunk_s|sample_kernel|verify_|probs_kernel|retrieval_|kv_write|shard_merge|correct_token|norm_prep|graph_step'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --gen 16 --profile-only > gpurun_out/ncu_launch.log 2>&1
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
$NCU -k regex:gemv_tc_kernel -s 51 -c 1 -o gpurun_out/ncu_wqkv -f python tools/ncu_targets.py retrieval > gpurun_out/ncu_wqkv.log 2>&1
$NCU -k regex:gemv_tc_kernel -s 52 -c 1 -o gpurun_out/ncu_wo -f python tools/ncu_targets.py retrieval > gpurun_out/ncu_wo.log 2>&1
$NCU -k regex:gemv_tc_kernel -s 53 -c 1 -o gpurun_out/ncu_wgu -f python tools/ncu_targets.py retrieval > gpurun_out/ncu_wgu.log 2>&1
$NCU -k regex:gemv_tc_kernel -s 54 -c 1 -o gpurun_out/ncu_wdown -f python tools/ncu_targets.py retrieval > gpurun_out/ncu_wdown.log 2>&1
SAN_TESTS="tests/test_gpu_kernels.py tests/test_gpu_session.py::test_forward_randomized_configs_match_oracle tests/test_gpu_session.py::test_draft_step_graphs_match_direct_forwards" SAN_K="gemv_tc or randomized or graphs" bash tools/gpu_sanitize.sh
ls gpurun_out/*.ncu-rep
exit 0
