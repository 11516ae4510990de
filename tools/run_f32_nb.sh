# adaLN GEMM (fp32 epilogue writes global directly): no staging buffers (def: 4 operand stages) vs 64 KB unused (prev: 3)
O=${O:-gpurun_out/f32}; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_dit_forward.py tests/test_gpu_dit_ops.py -m gpu -q > $O/tests.log 2>&1; tail -1 $O/tests.log
for v in def prev; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  env $L timeout 200 python tools/bits_step.py > $O/bits_$v.txt 2>&1; tail -1 $O/bits_$v.txt
  env $L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm -c 26 --csv python tools/ncu_step.py --steps 3 > $O/ncu_$v.csv 2>/dev/null
  python - $O/ncu_$v.csv $v <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
if rows:
    h = rows[0]; iv = h.index("Metric Value"); ik = h.index("Kernel Name")
    print(sys.argv[2], [r[iv] for r in rows[1:] if "256, 0" in r[ik]])
PY
done
