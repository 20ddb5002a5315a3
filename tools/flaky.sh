# repeat the GPU suite to catch intermittent failures; log failing test ids
for i in $(seq 1 ${N:-6}); do timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | grep -E "passed|FAILED|Error" | tail -3 >> gpurun_out/flaky.log; done
