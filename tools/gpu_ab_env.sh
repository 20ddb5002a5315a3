# Same-box A/B of environment switches through the bench, interleaved.
# ABENV="NAME=ENV1=v1,ENV2=v2;NAME2=" -> gpurun_out/abe_*.json
IFS=';' read -ra CASES <<< "$ABENV"
for rep in 1 2; do
  for c in "${CASES[@]}"; do
    name=${c%%=*}; envs=${c#*=}; [ "$envs" = "$c" ] && envs=""
    env $(echo "$envs" | tr "," " ") timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null > gpurun_out/abe_${name}_$rep.json
    python -c "import json; d=json.load(open('gpurun_out/abe_${name}_$rep.json')); print('$name', $rep, round(d['ms_per_token'],4), d['forward_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'], round(d['roofline']['avg_launch_us'],1))"
  done
done
exit 0
