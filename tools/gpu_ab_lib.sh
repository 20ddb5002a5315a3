# Same-box A/B of two library builds through the bench: A = ab/libhs_b200_A.so
# (an older build), B = the in-tree library.  Interleaved runs.  -> gpurun_out/abl_*.json
rm -rf /tmp/A && mkdir -p /tmp/A && cp -r . /tmp/A/ 2>/dev/null
cp ab/libhs_b200_A.so /tmp/A/paper_2404_11912_b200/libhs_b200.so
for rep in 1 2; do
  for arm in A B; do
    if [ $arm = A ]; then d=/tmp/A; else d=.; fi
    (cd $d && timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} 2>/dev/null) > gpurun_out/abl_${arm}_$rep.json
    python -c "import json,sys; d=json.load(open('gpurun_out/abl_${arm}_$rep.json')); print('$arm', $rep, round(d['ms_per_token'],4), d['forward_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['roofline']['avg_launch_us'],1))"
  done
done
exit 0
