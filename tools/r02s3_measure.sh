#!/bin/bash
# Round-2 (session 3) evidence batch (run under gpurun): bench lines, sweeps, launch list, ncu summaries.
set -u
O=${O:-gpurun_out/r02s3}
mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --model xl2 --no-decode > $O/bench_xl2.json 2> $O/bench_xl2.err
for n in 4 2 1; do
  timeout 200 python bench.py --guidance 7.5 --n $n --no-cpu-baseline --no-decode > $O/cfg_w7.5_n$n.json 2> $O/cfg_w7.5_n$n.err
done
for S in 1 2 4 8 64; do
  timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/streams_$S.json 2> $O/streams_$S.err
done
STEP="python tools/ncu_step.py --steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $STEP > /dev/null 2>&1
python tools/summarize_launches.py $O/launches.csv > $O/launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_tail|attn|gemm|patch|final" -s 3 -c 6 -o $O/ncu_full -f $STEP > $O/ncu_full.log 2>&1
python tools/ncu_summary.py $O/ncu_full.ncu-rep > $O/ncu_summary.md 2>&1
ls -la $O
