# ncu duration of the final-layer kernel for build variants (VARIANTS) and the default build
O=${O:-gpurun_out/fin}; mkdir -p $O
for v in def $VARIANTS; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:patch_embed -c 3 --csv python tools/ncu_step.py --steps 3 2>/dev/null | grep patch_embed | awk -F'","' '{print "'$v'", $(NF-2), $NF}' | tr -d '"'
done
