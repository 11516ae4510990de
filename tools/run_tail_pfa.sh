# Block tail: L2 prefetch of the next tile's attention rows (pa: at fc2 chunk 2/6/10; par6: + residual rows) vs none
O=${O:-gpurun_out/tpa}; mkdir -p $O
for v in def pa2 pa6 pa10 par6; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; echo "$v $(tail -1 $O/bits_$v.txt)"
done
for r in 1 2; do for v in def pa2 pa6 pa10 par6; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  echo -n "$v tail: "; env $L timeout 120 python tools/tail_bench.py --iters 20 2>&1 | tail -1
done; done
for r in 1 2; do for v in def pa2 pa6 pa10 par6; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/b_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_${v}_$r.json')); print('$v', round(d['value'],1), d['kernels']['block_tail'], d['clocks']['sm_mhz'])"
done; done
