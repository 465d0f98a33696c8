# The GPU test suite against the bounds-checked build (compute-sanitizer is not
# available on the GPU pool): every kernel's indices checked, a violation traps.
export OSP_LIB_VARIANT=checked
python -c "from paper_2306_16926_b200 import _capi; print(_capi.LIB_PATH)"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_codec.py -x -q 2>&1 | tail -3 > gpurun_out/r2_checked_parity.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -k oversub 2>&1 | tail -3 > gpurun_out/r2_checked_multi.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "resnet152" 2>&1 | tail -3 > gpurun_out/r2_checked_fullsize.log
timeout 300 python __graft_entry__.py > gpurun_out/r2_checked_smoke.log 2>&1
cat gpurun_out/r2_checked_*.log
