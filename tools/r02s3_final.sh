#!/bin/bash
# Final session-3 evidence: GPU tests, headline bench, S=1, XL, launch list, ncu of the top kernels
# and the two HBM kernels.
set -u
O=${O:-gpurun_out/r02s3c}
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --streams 1 --no-cpu-baseline --no-decode > $O/streams_1.json 2> $O/streams_1.err
timeout 300 python bench.py --model xl2 --no-decode > $O/bench_xl2.json 2> $O/bench_xl2.err
STEP="python tools/ncu_step.py --steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $STEP > /dev/null 2>&1
python tools/summarize_launches.py $O/launches.csv > $O/launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_tail|attn|gemm|patch|final" -s 3 -c 6 -o $O/ncu_full -f $STEP > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/ncu_full.ncu-rep > $O/ncu_summary.md 2>&1
ncu --set full --clock-control none -k regex:"patch_embed|final_layer" -c 2 -o $O/ncu_hbm -f $STEP > $O/ncu_hbm.log 2>&1
python tools/ncu_summary.py $O/ncu_hbm.ncu-rep > $O/ncu_hbm.md 2>&1
ls -la $O
