#!/bin/bash
# Closing evidence: full GPU suite, the default bench line, and the ncu launch list of bench.py
# itself (graph replay, as the driver runs it; -c bounds the capture)
set -u
O=${O:-gpurun_out/r02s3e}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
python -c "import json; d=json.load(open('$O/bench_default.json')); print(d['value'], d['e2e']['value'], d['clocks'])"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-decode > $O/bench_under_ncu.log 2>&1
python tools/summarize_launches.py $O/bench_launches.csv > $O/bench_launches.txt 2>&1
head -12 $O/bench_launches.txt
