# Patch embed: unrolled prologue (def) vs HEAD (prev), and 8 warps x 1 CTA/SM (w8)
O=${O:-gpurun_out/pe10}; mkdir -p $O
for v in def prev w8; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
done
for r in 1 2; do for v in def prev w8; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v" $(grep patch_embed $O/ncu_$v.csv | awk -F'","' '{print $NF}' | tr -d '"')
done; done
ncu --set full --clock-control none --import-source on -k regex:patch_embed -s 1 -c 1 -o $O/full_def -f python tools/ncu_step.py --steps 2 > /dev/null 2>&1
ncu -i $O/full_def.ncu-rep --page source --csv --print-source sass > $O/src_def.csv 2>&1
