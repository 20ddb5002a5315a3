# the other BASELINE configurations through the bench harness -> gpurun_out/cfg_*.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
run() { name=$1; shift; timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/cfg_$name.json 2> gpurun_out/cfg_$name.err;
  python -c "import json; d=json.load(open('gpurun_out/cfg_$name.json')); print('$name', round(d['ms_per_token'],3), d['acceptance'], round(d['step_roofline']['frac'],3), d.get('ar_ms_per_token'), d['clocks']['sm_mhz'])"; }
run 7b_T06 --temperature 0.6 --steps 6
run 13b_T06 --model llama2-13b --temperature 0.6 --steps 6
run lwm_262k --model lwm-7b --context 262144 --steps 6
run 7b_960 --steps 30
exit 0
