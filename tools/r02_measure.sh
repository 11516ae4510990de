#!/bin/bash
# Round-2 evidence batch (run under gpurun): bench lines, configs[2]/[3] sweeps, ncu, sanitizers.
set -u
O=gpurun_out/r02
mkdir -p $O
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python bench.py --model xl2 --no-decode > $O/bench_xl2.json 2> $O/bench_xl2.err
for n in 4 2 1; do
  timeout 200 python bench.py --guidance 7.5 --n $n --no-cpu-baseline --no-decode > $O/cfg_w7.5_n$n.json 2>&1
done
for n in 2 1; do
  timeout 200 python bench.py --n $n --no-cpu-baseline --no-decode > $O/cfg_w1_n$n.json 2>&1
done
for S in 64; do
  timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/streams_$S.json 2>&1
done
STEP="python tools/ncu_step.py --steps 2"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $STEP > /dev/null 2>&1
python tools/summarize_launches.py $O/launches.csv > $O/launches.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_tail|attn|gemm|patch|final" -s 3 -c 5 -o $O/ncu_full -f $STEP > $O/ncu_full.log 2>&1
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_step.py > $O/san_race.log 2>&1
echo "racecheck rc=$?" >> $O/san_race.log
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_step.py > $O/san_mem.log 2>&1
echo "memcheck rc=$?" >> $O/san_mem.log
ls -la $O
