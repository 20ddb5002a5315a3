# retrieval-view attention ring depth A/B, chunk_score pow2 mean
timeout 600 python tools/scorebench.py > gpurun_out/scorebench.json 2>&1; cat gpurun_out/scorebench.json | head -14
for d in 0 1; do echo "deep $d"; HS_ATT_DEEP=$d timeout 300 python tools/fwdbench.py --ctx 16384 --reps 10 2>&1 | tail -1; done
HS_ATT_DEEP=1 timeout 300 python tools/kbench.py --layers 4 --only attn 2>&1 | tail -12
HS_NVCC_DEFINES="-DAT_DEEP_K=3 -DAT_DEEP_V=3" python paper_2404_11912_b200/build.py --force > /dev/null 2>&1
echo "deep 3/3"; HS_ATT_DEEP=1 timeout 300 python tools/fwdbench.py --ctx 16384 --reps 10 2>&1 | tail -1
HS_NVCC_DEFINES="-DAT_DEEP_K=2 -DAT_DEEP_V=3" python paper_2404_11912_b200/build.py --force > /dev/null 2>&1
echo "deep 2/3"; HS_ATT_DEEP=1 timeout 300 python tools/fwdbench.py --ctx 16384 --reps 10 2>&1 | tail -1
exit 0
