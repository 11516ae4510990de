# compute-sanitizer on the session-3 kernels (run under gpurun)
O=${O:-gpurun_out/san}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_step.py > $O/memcheck_s2.log 2>&1; echo "rc=$?" >> $O/memcheck_s2.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_step.py --guidance 3 --streams 5 > $O/memcheck_s2_cfg.log 2>&1; echo "rc=$?" >> $O/memcheck_s2_cfg.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_step.py --xl --streams 1 --steps 1 > $O/memcheck_xl.log 2>&1; echo "rc=$?" >> $O/memcheck_xl.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_step.py > $O/racecheck_s2.log 2>&1; echo "rc=$?" >> $O/racecheck_s2.log
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_step.py > $O/synccheck_s2.log 2>&1; echo "rc=$?" >> $O/synccheck_s2.log
for f in $O/*.log; do echo "== $f"; tail -4 $f; done
