timeout 600 python tools/hostprof.py > gpurun_out/hostprof.txt 2>&1; head -60 gpurun_out/hostprof.txt | tail -45
bash tools/gpu_sanitize.sh
exit 0
