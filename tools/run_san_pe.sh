# compute-sanitizer on the patch-embed kernel after the copy-out / prologue changes
O=${O:-gpurun_out/san3}; mkdir -p $O
export PATH=/usr/local/cuda/bin:$PATH
K="--kernel-name kns=patch_embed"
timeout 600 compute-sanitizer --tool memcheck $K python tools/sanitize_step.py > $O/memcheck_pe_s2.log 2>&1; echo "rc=$?" >> $O/memcheck_pe_s2.log
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard $K python tools/sanitize_step.py > $O/racecheck_pe_s2.log 2>&1; echo "rc=$?" >> $O/racecheck_pe_s2.log
timeout 600 compute-sanitizer --tool synccheck $K python tools/sanitize_step.py > $O/synccheck_pe_s2.log 2>&1; echo "rc=$?" >> $O/synccheck_pe_s2.log
timeout 600 compute-sanitizer --tool memcheck $K python tools/sanitize_step.py --xl --streams 1 --steps 1 > $O/memcheck_pe_xl.log 2>&1; echo "rc=$?" >> $O/memcheck_pe_xl.log
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard $K python tools/sanitize_step.py --xl --streams 1 --steps 1 > $O/racecheck_pe_xl.log 2>&1; echo "rc=$?" >> $O/racecheck_pe_xl.log
for f in $O/*.log; do echo "== $f"; tail -3 $f; done
