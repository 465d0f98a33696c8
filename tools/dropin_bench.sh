#!/bin/bash
# Drop-in comparison at full model size: oracle/ref_driver.cpp built twice —
# against the reference engines (oracle/_ref/ref_driver) and against the B200
# façade (oracle/_ref/dropin_driver, Makefile.dropin) — runs the same
# synchronous OspWorker/OspServer message flow through the reference's own
# C++ API (host vectors in and out, as a reference user's code does).
#   golden: every per-iteration artefact of both builds compared byte for byte
#   bench : step time of both (1 host thread for the reference engine)
# Output: gpurun_out/dropin_bench.txt
set -u
mkdir -p gpurun_out
out=gpurun_out/dropin_bench.txt
: > $out
df -h /tmp | tail -1 >> $out
for layout in ${LAYOUTS:-resnet50 resnet152}; do
  # a full-size dump is ~9.4 GB per iteration for VGG-16 (rows of 8 workers x2):
  # 2 iterations there, and each layout's dumps are deleted after the compare
  iters=3; [ "$layout" = "vgg16" ] && iters=2
  lf=/tmp/osp_layers_$layout.txt
  python -c "from paper_2306_16926_b200 import layouts; print(','.join(map(str, layouts.get('$layout'))))" > $lf
  args="--layers-file $lf --workers 8 --budget-frac 0.5 --chunks 4 --seed 11"
  rm -rf /tmp/g_ref /tmp/g_dev; mkdir -p /tmp/g_ref /tmp/g_dev
  timeout 900 oracle/_ref/ref_driver golden $args --iters $iters --out /tmp/g_ref > /dev/null
  timeout 900 oracle/_ref/dropin_driver golden $args --iters $iters --out /tmp/g_dev > /dev/null
  nf=0; nd=0
  for f in /tmp/g_ref/*.bin; do
    nf=$((nf+1)); cmp -s "$f" "/tmp/g_dev/$(basename $f)" || { nd=$((nd+1)); echo "  differs: $(basename $f)" >> $out; }
  done
  echo "$layout golden: $nf files, $nd differ ($iters iterations, reference engines vs façade)" >> $out
  rm -rf /tmp/g_ref /tmp/g_dev
  r=$(timeout 900 oracle/_ref/ref_driver bench $args --iters 3 --warmup 1 --threads 1 | tail -1)
  d=$(timeout 900 oracle/_ref/dropin_driver bench $args --iters 5 --warmup 2 --threads 1 | tail -1)
  echo "$layout reference engines (CPU, 1 thread): $r" >> $out
  echo "$layout façade engines (B200, same API/flow): $d" >> $out
done
cat $out
