# chain: timing after the fence change + ncu of each role alone (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag10.txt; }
: > gpurun_out/r2_chain_diag10.txt
export OSP_SHARD_SYNC=chain
VAR=mixed run 29731 2 resnet50
cut -c1-300 gpurun_out/r2_chain_diag10.txt
timeout 600 ncu --set full --import-source on --target-processes all -k regex:k_shard_chain --launch-skip 4 -c 4 -f -o gpurun_out/r2_chain_solo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29732 tools/chain_solo.py > gpurun_out/r2_chain_ncu.log 2>&1; echo ncu=$?
tail -5 gpurun_out/r2_chain_ncu.log
ls -la gpurun_out/*.ncu-rep
