# streaming shard kernel variants (diagnostic): tile x ring x role split x mode at P (default 2)
for tile in ${TILES:-1024 2048}; do
for ks in ${KSS:-2}; do
for ae in ${AES:-2}; do
for mode in ${MODES:-1}; do
  echo "tile=$tile ks=$ks a_every=$ae mode=$mode"
  TILE=$tile OSP_SS_KS=$ks OSP_SS_AEVERY=$ae OSP_SS_MODE=$mode timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${P:-2} \
    --master-addr 127.0.0.1 --master-port 29611 tools/shard_diag.py ${LAYOUT:-resnet50} 20 2>&1 | grep -v "^\*\|OMP_NUM\|NCCL version\|Warning" | grep -A6 "rank 0"
done; done; done; done
