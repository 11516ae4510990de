# block tail tests + A/B timing against build_old
O=${O:-gpurun_out/tl1}; mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_bench_shape.py tests/test_gpu_dit_ops.py tests/test_gpu_dit_forward.py tests/test_gpu_stream_dit.py -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
for i in 1 2 3; do
  echo -n "old: "; SF_LIB_PATH=build_old/libstreamflow.so timeout 120 python tools/tail_bench.py --iters 20 2>&1 | tail -1
  echo -n "new: "; timeout 120 python tools/tail_bench.py --iters 20 2>&1 | tail -1
done
for v in old new; do
  if [ $v = old ]; then L="SF_LIB_PATH=build_old/libstreamflow.so"; else L=""; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/b_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_$v.json')); print('$v', round(d['value'],1), d['ms_per_step'], d['kernels']['block_tail'], d['clocks']['sm_mhz'])"
done
