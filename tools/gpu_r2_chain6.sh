# chain form: APPLY items alone vs PRE/FIN alone (2 GPUs)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag6.txt; }
: > gpurun_out/r2_chain_diag6.txt
: > gpurun_out/r2_diag.err
export OSP_SHARD_SYNC=chain
VAR=solo_apply OSP_SHARD_SOLO=apply run 29711 2 resnet50
VAR=solo_apply_pre1 OSP_SHARD_CHAIN_PRE=1 OSP_SHARD_SOLO=apply run 29712 2 resnet50
VAR=solo_apply_vgg OSP_SHARD_SOLO=apply run 29713 2 vgg16
VAR=solo_prefin_vgg run 29714 2 vgg16
cut -c1-400 gpurun_out/r2_chain_diag6.txt; grep -i -E "error|Traceback" gpurun_out/r2_diag.err | head
