# Patch embed: bit-identity against the previous build (build_prev) + ncu durations
O=${O:-gpurun_out/pe8}; mkdir -p $O
for v in def prev; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 120 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L timeout 120 python tools/bits_step.py --streams 5 --guidance 4.0 >> $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 >> $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v"; grep patch_embed $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | grep time
done
timeout 300 python -m pytest tests -m gpu -q -x -k "dit or stream or patch or xl or bench_shape" > $O/tests.log 2>&1; tail -1 $O/tests.log
