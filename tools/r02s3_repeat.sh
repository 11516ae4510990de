#!/bin/bash
# Run-to-run spread of the headline line (5 back-to-back default runs) + the reference arm
O=${O:-gpurun_out/rep}; mkdir -p $O
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-cpu-baseline --no-decode > $O/run_$i.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/run_$i.json')); print($i, round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['roofline']['frac'])"
done
timeout 900 python bench.py --impl reference > $O/reference.json 2> $O/reference.err
python -c "import json; d=json.load(open('$O/reference.json')); print('reference', d['value'], d.get('cpu_baseline',{}).get('cores'), d['config'].get('streams_total'))"
