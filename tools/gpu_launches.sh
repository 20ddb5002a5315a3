# ncu launch list (per-kernel durations) of a short bench run -> gpurun_out/launches.csv
KRE=${KRE:-'regex:attn_|gemv_|split_rows|rope_append|embed_kernel|chunk_s|sample_kernel|verify_|probs_kernel|retrieval_|kv_write|shard_merge|correct_token|norm_prep'}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" -c ${NCU_C:-4000} --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --gen 16 --profile-only > gpurun_out/ncu_launch.log 2>&1
python tools/launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; cat gpurun_out/launches_summary.txt | head -40
