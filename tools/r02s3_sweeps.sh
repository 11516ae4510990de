#!/bin/bash
# Closing sweeps on the final build: configs[2] CFG grid, configs[1]/[4] stream counts, XL, mock
set -u
O=${O:-gpurun_out/r02s3f}
mkdir -p $O
for n in 4 2 1; do
  timeout 200 python bench.py --guidance 7.5 --n $n --no-cpu-baseline --no-decode > $O/cfg_w7.5_n$n.json 2> $O/cfg_w7.5_n$n.err
done
for S in 1 2 4 8 64; do
  timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/streams_$S.json 2> $O/streams_$S.err
done
timeout 300 python bench.py --model xl2 --no-decode > $O/bench_xl2.json 2> $O/bench_xl2.err
timeout 600 python bench.py --model mock > $O/bench_mock_f64.json 2> $O/bench_mock_f64.err
for f in $O/*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d.get('p50_latency_ms') or 0,2), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
