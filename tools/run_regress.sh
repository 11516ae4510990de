# Same-box regression check of the headline: current build (def) vs the closing-evidence commit (base), interleaved
O=${O:-gpurun_out/reg}; mkdir -p $O
for r in 1 2 3; do for v in def base; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/b_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_${v}_$r.json')); print('$v', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
