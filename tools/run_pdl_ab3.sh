# PDL (small batches only, gated in-kernel by an argument) vs HEAD before PDL: S=32 alternated, S=1, S=4
O=${O:-gpurun_out/pdl3}; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
for i in 1 2 3; do
for v in nopdl new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --steps 60 --no-cpu-baseline --no-decode > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('S=32 $v', round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
done
for S in 1 2 4; do
for v in nopdl new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('S=$S $v', round(d['value'],1), round(d['ms_per_step'],4), round(d['p50_latency_ms'],3), d['clocks']['sm_mhz'])"
done
done
