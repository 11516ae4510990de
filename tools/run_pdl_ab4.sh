# standalone kernel A/B: HEAD before PDL vs now
for i in 1 2; do
for v in nopdl new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  echo "== $v"
  env $L timeout 120 python tools/tail_bench.py --iters 20 2>&1 | tail -1
  env $L timeout 120 python tools/attn_bench.py 2>&1 | head -1
  env $L timeout 120 python tools/gemm_bench.py 2>&1 | head -1
done
done
for v in nopdl new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --steps 60 --no-cpu-baseline --no-decode > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$v', round(d['value'],1), {a: b['ms_per_step'] for a, b in d['kernels'].items() if b['launches']})"
done
