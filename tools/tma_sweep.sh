# TMA-staged stage kernels: tile / ring-shape sweep (diagnostic, one GPU)
python tools/tma_compare.py --variants reg-512,tma-512,tma-1024,tma-2048 --layouts resnet50,resnet152,vgg16,llama1b
for ks in 2 3; do
OSP_TMA_CW=4 OSP_TMA_STAGES=$ks timeout 120 python tools/tma_compare.py --variants tma-512,tma-1024,tma-2048 --layouts resnet50 2>&1 | grep -E "step|Error"
done
