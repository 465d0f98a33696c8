# single-launch step: 1024 threads for many-tile layouts; parity at both sizes, MLP lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small" 2>&1 | tail -1
OSP_SMALL_THREADS=1024 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "small" 2>&1 | tail -1
for L in mlp mlp_acc; do for TH in 512 1024; do OSP_SMALL_THREADS=$TH timeout 300 python bench.py --layout $L --steps 3200 --warmup 32 --graph --no-cpu-baseline --overlap-ms 0 --e2e-steps 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$L', $TH, round(d['ms_per_step']*1e3,2), 'us')"; done; done
