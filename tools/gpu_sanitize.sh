# compute-sanitizer (memcheck, racecheck, synccheck) over the kernel tests -> gpurun_out/sanitize_*.log
S=gpurun_out
K="${SAN_K:-attention or gemv_tc or gemm3 or build or score or sampling or verify or combine}"
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_T:-900} compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python -m pytest tests/test_gpu_kernels.py -q -x -k "$K" > $S/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $S/sanitize_$tool.log
done
exit 0
