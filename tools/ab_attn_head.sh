# attention A/B: current build vs build_head (HEAD), + attention parity tests
timeout 300 python -m pytest tests/test_gpu_dit_ops.py tests/test_gpu_dit_forward.py tests/test_gpu_dit_xl.py tests/test_gpu_bench_shape.py -x -q 2>&1 | tail -1
for i in 1 2 3; do
  echo -n "head "; SF_LIB_PATH=build_head/libstreamflow.so timeout 120 python tools/attn_bench.py 2>&1 | head -1
  echo -n "new  "; timeout 120 python tools/attn_bench.py 2>&1 | head -1
done
for v in head new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-decode > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$v', round(d['value'],1), d['kernels']['attention'], d['clocks']['sm_mhz'])"
done
