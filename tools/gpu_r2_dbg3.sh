mkdir -p gpurun_out; : > gpurun_out/r2_dbg3.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "lagging" 2>&1 | tail -3 >> gpurun_out/r2_dbg3.log
for i in $(seq 1 8); do timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "oversubscribed_ragged" > /tmp/o.txt 2>&1; if grep -q failed /tmp/o.txt; then echo "RUN $i FAILED" >> gpurun_out/r2_dbg3.log; grep -E "AssertionError|FAILED" /tmp/o.txt | head -10 >> gpurun_out/r2_dbg3.log; else echo "run $i ok" >> gpurun_out/r2_dbg3.log; fi; done
cat gpurun_out/r2_dbg3.log
