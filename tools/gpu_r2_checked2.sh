# the bounds-checked build over the round-2 additions (chain form, learner, pipelined host step)
export OSP_LIB_VARIANT=checked
mkdir -p gpurun_out
python -c "from paper_2306_16926_b200 import _capi; print(_capi.LIB_PATH)"
timeout 900 python -m pytest tests/test_gpu_learner.py -x -q 2>&1 | tail -1 > gpurun_out/r2_checked2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "step_host or small" 2>&1 | tail -1 >> gpurun_out/r2_checked2.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -k "oversub or ties or lagging" 2>&1 | tail -1 >> gpurun_out/r2_checked2.log
cat gpurun_out/r2_checked2.log
