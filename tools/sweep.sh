#!/bin/bash
# BASELINE configs[2] (CFG x 1/2/4-step grids) and the per-GPU share of configs[4]
# (64-512 streams over 8 GPUs = 8-64 streams per GPU), one bench line each.
OUT=${OUT:-gpurun_out/sweep.jsonl}
: > $OUT
for args in "--guidance 7.5 --n 4" "--guidance 7.5 --n 2" "--guidance 7.5 --n 1" "--n 2" "--n 1" \
            "--streams 8" "--streams 16" "--streams 64"; do
  timeout 300 python bench.py $args --steps 20 --warmup 4 --no-cpu-baseline --no-decode 2>/dev/null | tail -1 >> $OUT
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    c = d["config"]
    print(f'w={c["guidance_scale"]} n={c["steps_per_generation"]} S={c["streams_per_gpu"]}: {d["value"]:8.1f} frames/s, '
          f'{d["ms_per_step"]:6.2f} ms/step, p50 {d["p50_latency_ms"]:6.2f} ms, p99 {d["p99_latency_ms"]:6.2f} ms, '
          f'step {d["step_roofline"]["frac"]:.3f} of sustained')
PY
