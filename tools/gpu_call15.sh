for st in 5 10; do
  HS_NVCC_DEFINES="-DHS_TC_STAGES=$st" python paper_2404_11912_b200/build.py --force > /dev/null 2>&1
  echo "stages $st"; timeout 300 python tools/kbench.py --layers 4 --only w 2>&1 | python -c "
import sys,json
txt=sys.stdin.read(); i=txt.find('{'); d=json.loads(txt[i:])
print({k:(round(v['us'],2), round(v['GBps'])) for k,v in d['gemv'].items() if k.endswith('_t3')})"
done
exit 0
