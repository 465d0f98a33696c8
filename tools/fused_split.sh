# barrier-mode fused apply1 || agg2 warp split (diagnostic): OSP_FUSED_APPLY_EVERY at P ranks
for e in ${ES:--4}; do
  OSP_FUSED_APPLY_EVERY=$e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${P:-2} \
    --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus ${P:-2} --steps 100 --e2e-steps 1 --overlap-ms 0 2>&1 \
    | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('P=${P:-2} apply_every=$e', round(d['ms_per_step'],4), {k: round(v, 4) for k, v in d['phase_ms'].items()})"
done
