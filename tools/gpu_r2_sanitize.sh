# compute-sanitizer over every kernel family + the drop-in façade flow at full size
bash tools/sanitize.sh > gpurun_out/r2_sanitize_summary.txt 2>&1
LAYOUTS="resnet50 vgg16" bash tools/dropin_bench.sh > /dev/null 2>&1
cat gpurun_out/r2_sanitize_summary.txt gpurun_out/dropin_bench.txt
for f in gpurun_out/sanitize_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|sanitize .*ok|Error|error" $f | head -5; done
