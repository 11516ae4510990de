# DiT-XL/2 GEMM tests + XL bench A/B against build_old
O=${O:-gpurun_out/xl1}; mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_dit_xl.py tests/test_gpu_stream_dit.py tests/test_gpu_dit_ops.py -x -q > $O/tests.log 2>&1; tail -2 $O/tests.log
for v in old new; do
  if [ $v = old ]; then L="SF_LIB_PATH=build_old/libstreamflow.so"; else L=""; fi
  env $L timeout 300 python bench.py --model xl2 --no-cpu-baseline --no-decode > $O/xl_$v.json 2> $O/xl_$v.err
  python -c "import json; d=json.load(open('$O/xl_$v.json')); k=d['kernels']; print('$v', round(d['value'],1), round(d['ms_per_step'],3), {a: b['ms_per_step'] for a, b in k.items() if b['launches']}, d['clocks'])"
done
