O=${O:-gpurun_out/g1}; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -2 $O/tests.log
for S in 32 1; do
timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/bench_S$S.json 2> $O/bench_S$S.err
python -c "import json; d=json.load(open('$O/bench_S$S.json')); k=d['kernels']; print($S, d['value'], d['ms_per_step'], d.get('p50_latency_ms'), {a: b['ms_per_step'] for a, b in k.items() if b['launches']}, d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --model xl2 --no-cpu-baseline --no-decode > $O/bench_xl2.json 2> $O/bench_xl2.err
python -c "import json; d=json.load(open('$O/bench_xl2.json')); print('xl2', d['value'], d['ms_per_step'])"
