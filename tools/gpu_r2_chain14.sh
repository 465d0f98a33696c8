# chain form: bounded PRE lead (keep the running sums in L2 until the next rank pulls them)
mkdir -p gpurun_out
run() { OSP_SHARD_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $1 tools/shard_x_diag.py ${@:3} 2>>gpurun_out/r2_diag.err | tail -1 | sed "s/^/$VAR /" >> gpurun_out/r2_chain_diag15.txt; }
: > gpurun_out/r2_chain_diag15.txt
VAR=base run 29801 2 resnet50
VAR=max8 OSP_SHARD_CHAIN_MAXLEAD=8 run 29802 2 resnet50
VAR=max16 OSP_SHARD_CHAIN_MAXLEAD=16 run 29803 2 resnet50
VAR=max24 OSP_SHARD_CHAIN_MAXLEAD=24 run 29804 2 resnet50
VAR=base_b run 29805 2 resnet50
VAR=max16_vgg OSP_SHARD_CHAIN_MAXLEAD=16 run 29806 2 vgg16
VAR=base_vgg run 29807 2 vgg16
