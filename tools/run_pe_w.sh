# Patch embed: warps per CTA / CTAs per SM variants (ncu durations; bits of each)
O=${O:-gpurun_out/pe9}; mkdir -p $O
for v in def w14 w13 w4; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v"; grep patch_embed $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
