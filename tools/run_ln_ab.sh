# XL LayerNorm + modulate kernel variants: bits of the XL step, ncu durations
O=${O:-gpurun_out/ln1}; mkdir -p $O
for v in def prev c3 p2 t1; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ln_modulate -s 4 -c 6 --csv python tools/bits_step.py --xl --streams 2 --steps 1 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v" $(grep ln_modulate $O/ncu_$v.csv | awk -F'","' '{print $NF}' | tr -d '"')
done
timeout 300 python -m pytest tests/test_gpu_dit_xl.py -m gpu -q -x > $O/tests.log 2>&1; tail -1 $O/tests.log
