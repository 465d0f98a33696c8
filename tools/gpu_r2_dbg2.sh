mkdir -p gpurun_out; : > gpurun_out/r2_dbg2.log
for i in $(seq 1 14); do timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "oversubscribed_ragged" > /tmp/o.txt 2>&1; if grep -q failed /tmp/o.txt; then echo "RUN $i FAILED" >> gpurun_out/r2_dbg2.log; grep -E "AssertionError|assert |Error|rank|it [0-9]|FAILED|sync" /tmp/o.txt | head -40 >> gpurun_out/r2_dbg2.log; else echo "run $i ok" >> gpurun_out/r2_dbg2.log; fi; done
cat gpurun_out/r2_dbg2.log
