# One GPU call: kernel micro-bench, hot-path launch list, ncu --set full of
# the top kernels.  Outputs land in gpurun_out/ (copied to profiles/ by hand).
set -x
KRE='regex:attn_|gemv_|split_rows|rope_append|embed_kernel|chunk_s|sample_kernel|verify_|probs_kernel|retrieval_|kv_write|shard_merge|correct_token'
timeout 600 python tools/kbench.py --layers 4 --json gpurun_out/kbench.json > gpurun_out/kbench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c 4000 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --gen 16 --profile-only > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 4 -c 1 \
  -o gpurun_out/attn_tc_full -f python tools/kbench.py --layers 2 --only attn > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc_kernel -s 12 -c 1 \
  -o gpurun_out/gemv_tc_full -f python tools/kbench.py --layers 2 --only wgu > gpurun_out/ncu_gemv.log 2>&1
tail -3 gpurun_out/*.log
