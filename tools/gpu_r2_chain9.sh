# ncu of the chain form's roles alone: one rank under ncu, the other plain (2 GPUs)
mkdir -p gpurun_out
export OSP_SHARD_SYNC=chain MASTER_ADDR=127.0.0.1 WORLD_SIZE=2
for PR in 0 1; do
  OR=$((1 - PR))
  MASTER_PORT=2974$PR RANK=$OR LOCAL_RANK=$OR timeout 600 python tools/chain_solo.py > gpurun_out/r2_chain_plain$OR.log 2>&1 &
  MASTER_PORT=2974$PR RANK=$PR LOCAL_RANK=$PR timeout 600 ncu --set full --import-source on -k regex:k_shard_chain --launch-skip 4 -c 2 -f -o gpurun_out/r2_chain_solo_rank$PR python tools/chain_solo.py > gpurun_out/r2_chain_ncu$PR.log 2>&1
  echo ncu$PR=$?
  wait
  tail -3 gpurun_out/r2_chain_ncu$PR.log
done
ls -la gpurun_out/*.ncu-rep
