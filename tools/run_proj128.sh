# DiT-XL/2 attention projection (gated residual, K=1152): 128-wide pair tiles (p128: 288 tiles = 3.9 waves on 74 clusters) vs 192 (def: 2.6 waves)
O=${O:-gpurun_out/p128}; mkdir -p $O
SF_LIB_PATH=build_p128/libstreamflow.so timeout 300 python -m pytest tests/test_gpu_dit_xl.py tests/test_gpu_stream_dit.py -m gpu -q > $O/tests_p128.log 2>&1; tail -1 $O/tests_p128.log
for v in def p128; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 > $O/bits_$v.txt 2>&1; echo "$v $(tail -1 $O/bits_$v.txt)"
done
for r in 1 2; do for v in def p128; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --model xl2 --no-decode --no-cpu-baseline > $O/xl_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/xl_${v}_$r.json')); k=d['kernels']; print('$v', round(d['value'],1), k['proj_gemm_res_ln']['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
