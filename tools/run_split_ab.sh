# block-tail column split for small batches: parity tests + A/B against build_head
O=${O:-gpurun_out/split}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_bench_shape.py tests/test_gpu_dit_forward.py tests/test_gpu_stream_dit.py tests/test_gpu_multirank.py tests/test_gpu_dit_ops.py -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
for S in 1 2 32; do
for v in head new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('S=$S $v', round(d['value'],1), round(d['ms_per_step'],4), round(d['p50_latency_ms'],3), d['kernels']['block_tail'], d['clocks']['sm_mhz'])"
done
done
