#!/bin/bash
# ncu evidence for the bench workload (run under gpurun; one GPU).
#   launches.csv : every launch of 2 eager steps (gpu__time_duration, cold/serialised)
#   attn.ncu-rep : --set full on one attention launch
#   gemm.ncu-rep : --set full on the qkv/proj/fc1/fc2 GEMMs of layer 0
#   misc.ncu-rep : --set full on cond/patch-embed/final kernels
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-prof}
mkdir -p $OUT
STEP="python tools/ncu_step.py --steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $STEP > /dev/null 2>&1
python tools/summarize_launches.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn -s 2 -c 1 -o $OUT/${TAG}_attn -f $STEP > $OUT/${TAG}_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm -s 1 -c 4 -o $OUT/${TAG}_gemm -f $STEP > $OUT/${TAG}_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mlp_fused|block_tail" -s 1 -c 1 -o $OUT/${TAG}_mlp -f $STEP > $OUT/${TAG}_mlp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'cond_kernel|patch_embed|final_layer' -c 3 -o $OUT/${TAG}_misc -f $STEP > $OUT/${TAG}_misc.log 2>&1
ls -la $OUT
