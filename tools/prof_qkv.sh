# ncu --set full of layer 0's QKV GEMM in the bench step (+ raw and SASS-source pages)
set -u
O=${O:-gpurun_out/p2}
mkdir -p $O
STEP="python tools/ncu_step.py --steps 2"
ncu --set full --clock-control none --import-source on -k regex:gemm -s 1 -c 1 -o $O/qkv -f $STEP > $O/qkv.log 2>&1
ncu -i $O/qkv.ncu-rep --page raw --csv > $O/qkv_raw.csv 2>&1
ncu -i $O/qkv.ncu-rep --page source --csv --print-source sass > $O/qkv_src.csv 2>&1
