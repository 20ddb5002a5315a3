# A/B of experiment hooks on single lane forwards (tools/fwdbench.py, 7B shape).
# AB="NAME=ENV1=v1,ENV2=v2;NAME2=..."  Outputs -> gpurun_out/ab.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
: > gpurun_out/ab.jsonl
for rep in 1 2; do
IFS=';' read -ra CASES <<< "$AB"
for c in "${CASES[@]}"; do
  name=${c%%=*}; envs=${c#*=}
  [ "$envs" = "$c" ] && envs=""
  env $(echo "$envs" | tr "," " ") timeout 300 python tools/fwdbench.py --ctx ${CTX:-16384} --reps ${REPS:-20} > gpurun_out/ab_$name.out 2>&1; line=$(grep "^{" gpurun_out/ab_$name.out | tail -1)
  echo "{\"case\": \"$name\", \"rep\": $rep, \"r\": $line}" | tee -a gpurun_out/ab.jsonl
done
done
exit 0
