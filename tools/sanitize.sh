# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (smoke sizes). Logs under gpurun_out/sanitize_*.log.
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for kind in group register small; do
    timeout 900 $CS --tool $tool --error-exitcode 17 python tools/sanitize_step.py $kind \
      > gpurun_out/sanitize_${tool}_${kind}.log 2>&1
    echo "$tool $kind rc=$?"
  done
  # the sharded kernels: two ranks on one GPU (oversubscribed), both under the tool
  MASTER_ADDR=127.0.0.1 MASTER_PORT=29517 timeout 1200 $CS --tool $tool --error-exitcode 17 \
    --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 tools/sanitize_step.py shard \
    > gpurun_out/sanitize_${tool}_shard.log 2>&1
  echo "$tool shard rc=$?"
done
