# A/B of attention build variants (build_<name>/libstreamflow.so) at the bench shape, 2 rounds
for i in 1 2; do
for v in def $VARIANTS; do
  if [ $v = def ]; then L=""; else L="SF_LIB_PATH=build_$v/libstreamflow.so"; fi
  echo -n "$v: "; env $L timeout 120 python tools/attn_bench.py 2>&1 | head -1
done
done
