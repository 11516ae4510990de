# DiT-XL/2 gated-residual GEMM (192-wide pair tiles): 12 epilogue warps (def, 4 ring stages) vs 8 (r8, 5 stages)
O=${O:-gpurun_out/resw}; mkdir -p $O
SF_LIB_PATH=build_r8/libstreamflow.so timeout 300 python -m pytest tests/test_gpu_dit_xl.py tests/test_gpu_gemm.py -m gpu -q > $O/tests_r8.log 2>&1; tail -1 $O/tests_r8.log
for v in def r8; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"gemm_bf16_tcgen05<192" -s 4 -c 4 --csv python tools/bits_step.py --xl --streams 2 --steps 1 > $O/ncu_$v.csv 2>/dev/null
  echo "== $v" $(grep gemm_bf16 $O/ncu_$v.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | tr '\n' ' ')
done
for r in 1 2; do for v in def r8; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --model xl2 --no-decode --no-cpu-baseline > $O/xl_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/xl_${v}_$r.json')); k=d['kernels']; print('$v', round(d['value'],1), k['proj_gemm_res_ln']['ms_per_step'], k['fc2_gemm_res_ln']['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
