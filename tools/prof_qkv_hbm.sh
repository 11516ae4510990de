set -u
O=gpurun_out/p1
mkdir -p $O
STEP="python tools/ncu_step.py --steps 2"
ncu --set full --clock-control none --import-source on -k regex:gemm -s 1 -c 1 -o $O/qkv -f $STEP > $O/qkv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"patch|final" -c 2 -o $O/hbm -f $STEP > $O/hbm.log 2>&1
ncu -i $O/qkv.ncu-rep --page raw --csv > $O/qkv_raw.csv 2>&1
ncu -i $O/qkv.ncu-rep --page source --csv --print-source sass > $O/qkv_src.csv 2>&1
ncu -i $O/hbm.ncu-rep --page raw --csv > $O/hbm_raw.csv 2>&1
ncu -i $O/hbm.ncu-rep --page source --csv --print-source sass > $O/hbm_src.csv 2>&1
ls -la $O
