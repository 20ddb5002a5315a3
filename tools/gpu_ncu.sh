# ncu --set full captures of the retrieval-forward kernels and chunk_score (one launch each, warm)
# -> gpurun_out/ncu_*.ncu-rep (summarised into profiles/ by tools/ncu_summary.py)
S=gpurun_out
NCU="timeout 600 ncu --set full --clock-control none --import-source on"
# tools/ncu_targets.py retrieval: 6 forwards x (4 layers x 4 GEMVs + lm_head) = 17 GEMV launches per forward
$NCU -k regex:gemv_tc_kernel -s 51 -c 1 -o $S/ncu_wqkv -f python tools/ncu_targets.py retrieval > $S/ncu_wqkv.log 2>&1
$NCU -k regex:gemv_tc_kernel -s 52 -c 1 -o $S/ncu_wo -f python tools/ncu_targets.py retrieval > $S/ncu_wo.log 2>&1
$NCU -k regex:gemv_tc_kernel -s 53 -c 1 -o $S/ncu_wgu -f python tools/ncu_targets.py retrieval > $S/ncu_wgu.log 2>&1
$NCU -k regex:gemv_tc_kernel -s 54 -c 1 -o $S/ncu_wdown -f python tools/ncu_targets.py retrieval > $S/ncu_wdown.log 2>&1
$NCU -k regex:attn_tc_kernel -s 12 -c 1 -o $S/ncu_attn_retr -f python tools/ncu_targets.py retrieval > $S/ncu_attn_retr.log 2>&1
$NCU -k regex:attn_combine -s 12 -c 1 -o $S/ncu_combine_retr -f python tools/ncu_targets.py retrieval > $S/ncu_combine_retr.log 2>&1
$NCU -k regex:chunk_score -s 3 -c 1 -o $S/ncu_chunk_score -f python tools/ncu_targets.py score > $S/ncu_score.log 2>&1
[ -n "$GEMM" ] && $NCU -k regex:gemm3_tc -s 3 -c 1 -o $S/ncu_gemm3 -f python tools/gemmbench.py --reps 2 > $S/ncu_gemm3.log 2>&1
ls -la $S/*.ncu-rep; tail -2 $S/ncu_*.log
exit 0
