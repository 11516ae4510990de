# Patch embed: residual written by STG from the copy-out loop instead of a TMA store (variant stg)
O=${O:-gpurun_out/pe7}; mkdir -p $O
for v in def stg; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 >> $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
done
for r in 1 2; do for v in def stg; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L ncu --metrics gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v"; grep patch_embed $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | grep time
done; done
