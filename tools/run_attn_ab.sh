# attention tests + A/B timing against build_old (the previous kernel)
O=${O:-gpurun_out/at1}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dit_ops.py tests/test_gpu_dit_forward.py tests/test_gpu_dit_xl.py -x -q > $O/tests.log 2>&1; tail -2 $O/tests.log
for i in 1 2; do
  echo -n "old: "; SF_LIB_PATH=build_old/libstreamflow.so timeout 120 python tools/attn_bench.py 2>&1 | head -2 | tr '\n' ' '; echo
  echo -n "new: "; timeout 120 python tools/attn_bench.py 2>&1 | head -2 | tr '\n' ' '; echo
done
