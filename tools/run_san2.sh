O=${O:-gpurun_out/san2}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
for i in 1 2; do
  echo -n "old: "; SF_LIB_PATH=build_old/libstreamflow.so timeout 120 python tools/attn_bench.py 2>&1 | head -1
  echo -n "new: "; timeout 120 python tools/attn_bench.py 2>&1 | head -1
done
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_step.py > $O/synccheck_s2.log 2>&1; echo "rc=$?" >> $O/synccheck_s2.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_step.py --xl --streams 1 --steps 1 > $O/synccheck_xl.log 2>&1; echo "rc=$?" >> $O/synccheck_xl.log
for f in $O/*.log; do echo "== $f"; tail -3 $f; done
