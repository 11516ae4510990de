# programmatic dependent launch: tests + A/B at S = 1, 4, 32 against build_nopdl
O=${O:-gpurun_out/pdl1}; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
for S in 1 4 32; do
for v in nopdl new; do
  if [ $v = new ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --streams $S --no-cpu-baseline --no-decode > $O/b_${v}_$S.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_${v}_$S.json')); print('S=$S $v', round(d['value'],1), round(d['ms_per_step'],4), round(d['p50_latency_ms'],3), d['clocks']['sm_mhz'])"
done
done
