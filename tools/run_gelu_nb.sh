# DiT-XL/2 fc1 (GELU, 256-wide pair tiles, 16 epilogue warps): one staging buffer per warp (g1: 5 operand stages) vs two (def: 4)
O=${O:-gpurun_out/gnb}; mkdir -p $O
SF_LIB_PATH=build_g1/libstreamflow.so timeout 300 python -m pytest tests/test_gpu_dit_xl.py tests/test_gpu_gemm.py -m gpu -q > $O/tests_g1.log 2>&1; tail -1 $O/tests_g1.log
for v in def g1; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
done
for r in 1 2; do for v in def g1; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --model xl2 --no-decode --no-cpu-baseline > $O/xl_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/xl_${v}_$r.json')); k=d['kernels']; print('$v', round(d['value'],1), k['fc1_gemm_gelu']['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
