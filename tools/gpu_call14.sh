# GEMV ring depth vs isolated throughput (1 CTA/SM beyond 5 stages)
for st in 5 8 10 11; do
  HS_NVCC_DEFINES="-DHS_TC_STAGES=$st" python paper_2404_11912_b200/build.py --force > /dev/null 2>&1
  echo "stages $st"; timeout 300 python tools/kbench.py --layers 4 --only _t3 2>&1 | python -c "
import sys,json
txt=sys.stdin.read(); i=txt.find('{'); d=json.loads(txt[i:])
print({k:round(v['us'],2) for k,v in d['gemv'].items()})"
  timeout 300 python tools/fwdbench.py --ctx 16384 --reps 10 2>&1 | tail -1
done
exit 0
