# DiT-XL/2 QKV (head dim 72, 144-wide pair tiles): 4 epilogue warps (def) vs 8 = one head per warp (q8); prev = HEAD build
O=${O:-gpurun_out/q144}; mkdir -p $O
SF_LIB_PATH=build_q8/libstreamflow.so timeout 300 python -m pytest tests/test_gpu_dit_xl.py tests/test_gpu_gemm.py tests/test_gpu_stream_dit.py -m gpu -q > $O/tests_q8.log 2>&1; tail -1 $O/tests_q8.log
timeout 300 python -m pytest tests/test_gpu_dit_xl.py tests/test_gpu_gemm.py -m gpu -q > $O/tests_def.log 2>&1; tail -1 $O/tests_def.log
for v in def prev q8; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python tools/bits_step.py --xl --streams 2 > $O/bits_$v.txt 2>&1; echo "$v $(tail -1 $O/bits_$v.txt)"
done
for r in 1 2; do for v in def q8; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 300 python bench.py --model xl2 --no-decode --no-cpu-baseline > $O/xl_${v}_$r.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/xl_${v}_$r.json')); k=d['kernels']; print('$v', round(d['value'],1), k['qkv_gemm']['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
