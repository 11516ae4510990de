# Patch-embed split-unit kernel: parity tests, bits across variants, durations, one full capture
O=${O:-gpurun_out/pe6}; mkdir -p $O
timeout 300 python -m pytest tests -m gpu -q -x -k "dit or stream or patch or xl or bench_shape" > $O/tests.log 2>&1; tail -2 $O/tests.log
for v in def c3 oldpad; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L ncu --metrics gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v"; grep patch_embed $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
ncu --set full --clock-control none --import-source on -k regex:patch_embed -s 1 -c 1 -o $O/full_def -f python tools/ncu_step.py --steps 2 > /dev/null 2>&1
ncu -i $O/full_def.ncu-rep --page source --csv --print-source sass > $O/src_def.csv 2>&1
