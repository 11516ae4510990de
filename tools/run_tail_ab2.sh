# block tail A/B: current build vs build_early (projection loads right after a2full)
timeout 400 python -m pytest tests/test_gpu_bench_shape.py tests/test_gpu_dit_forward.py -x -q 2>&1 | tail -1
for i in 1 2 3; do
  echo -n "early: "; SF_LIB_PATH=build_early/libstreamflow.so timeout 120 python tools/tail_bench.py --iters 20 2>&1 | tail -1
  echo -n "new:   "; timeout 120 python tools/tail_bench.py --iters 20 2>&1 | tail -1
done
for v in early new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-decode > /tmp/b.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$v', round(d['value'],1), d['kernels']['block_tail'], d['clocks']['sm_mhz'])"
done
