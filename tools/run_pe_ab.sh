# Patch-embed rewrite: bit-identity against the previous kernel (HEAD build) + ncu duration of the variants
O=${O:-gpurun_out/pe4}; mkdir -p $O
for v in def old; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L timeout 120 python tools/bits_step.py --streams 5 --guidance 4.0 >> $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 >> $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
done
for v in def old c2 u12; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v"; grep patch_embed $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
timeout 300 python -m pytest tests -m gpu -q -x -k "dit or stream or patch or xl" > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 300 python bench.py --no-cpu-baseline --no-decode > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.load(open('$O/bench.json')); k=d['kernels']; print(d['value'], d['ms_per_step'], k['patch_embed_ln'], d['clocks']['sm_mhz'])"
