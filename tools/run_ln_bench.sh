# XL bench line with the new LN kernel (def) vs the previous build (prev), twice each
O=${O:-gpurun_out/ln2}; mkdir -p $O
for r in 1 2; do for v in def prev; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --model xl2 --no-decode --no-cpu-baseline > $O/xl_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/xl_${v}_$r.json')); k=d['kernels']; print('$v', round(d['value'],1), d['ms_per_step'], k['proj_gemm_res_ln'], k['fc2_gemm_res_ln'], d['clocks']['sm_mhz'])"
done; done
