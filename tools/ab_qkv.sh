mkdir -p gpurun_out/ab1
for i in 1 2; do
for v in def pf0 pf1 pf3; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  echo -n "$v: "; env $L timeout 120 python tools/gemm_bench.py 2>&1 | head -1
done
done
for v in def pf0; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-decode > gpurun_out/ab1/bench_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab1/bench_$v.json')); print('$v', d['value'], d['ms_per_step'], d['kernels']['qkv_gemm'], d['clocks']['sm_mhz'])"
done
