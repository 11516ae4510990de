# Conditioning kernels (8 rows per block) vs previous build; adaLN GEMM capture
O=${O:-gpurun_out/cd1}; mkdir -p $O
timeout 400 python -m pytest tests -m gpu -q -x -k "dit or stream or xl or bench_shape or cond" > $O/tests.log 2>&1; tail -1 $O/tests.log
for v in def prev; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  for S in 32 1; do
    env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cond_|gemm_bf16_tcgen05<256, 0" -c 6 --csv python tools/ncu_step.py --steps 2 --streams $S > $O/ncu_${v}_$S.csv 2>/dev/null
    echo "== $v S=$S"; grep -E "cond_|gemm" $O/ncu_${v}_$S.csv | awk -F'","' '{print $5, $NF}' | tr -d '"' | cut -c1-80
  done
done
ncu --set full --clock-control none --import-source on -k regex:"gemm_bf16_tcgen05<256, 0" -c 1 -o $O/ada -f python tools/ncu_step.py --steps 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/ada.ncu-rep > $O/ada.md 2>&1
ncu -i $O/ada.ncu-rep --page raw --csv > $O/ada_raw.csv 2>&1
timeout 300 python bench.py --streams 1 --no-cpu-baseline --no-decode > $O/s1.json 2>/dev/null
python -c "import json; d=json.load(open('$O/s1.json')); print('S=1', d['value'], d['ms_per_step'], d['p50_latency_ms'], d['kernels']['cond'], d['kernels']['adaln_gemm'])"
