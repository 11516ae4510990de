"""The reference-side ctypes binding of INTEGRATION.md section 3 (integration/flowpipe_b200.py),
installed into the UNMODIFIED reference package (baseline/_ref): flowpipe.run_stream with the
GPU Euler step must give the reference's own numpy results bit for bit (fp64 and fp32, with
and without CFG), and the binding must raise the reference's exceptions.  Runs in a subprocess
(tests/ref_suite aliases the name ``flowpipe`` to this package inside the pytest process)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, REF); sys.path.insert(0, ROOT)
import flowpipe
from integration import flowpipe_b200 as b200
sched = flowpipe.build_time_window_schedule(num_windows=3, inference_steps=4)
cases = []
for dt in (np.float64, np.float32):
    for w in (1.0, 7.5):
        model = flowpipe.SeededMockModel(dim=512, seed=3)
        cond = flowpipe.make_conditioning(embedding=np.linspace(-1, 1, 8), guidance_scale=w)
        cases.append((model, cond, dt))
ref = [flowpipe.run_stream(6, 4, m, c, 11, sched, dtype=dt) for m, c, dt in cases]
b200.install(flowpipe, LIB)
got = [flowpipe.run_stream(6, 4, m, c, 11, sched, dtype=dt) for m, c, dt in cases]
for (rr, rs), (gr, gs) in zip(ref, got):
    assert [r.id for r in rr] == [r.id for r in gr]
    for a, b in zip(rr, gr):
        assert a.latent.dtype == b.latent.dtype and np.array_equal(a.latent, b.latent), (a.id, np.abs(a.latent - b.latent).max())
    assert rs.step_stats.param_evals == gs.step_stats.param_evals and rs.scheduler_calls == gs.scheduler_calls
bad = flowpipe.velocity.LatentBatch(data=np.zeros((1, 4)), timesteps=np.array([0.3]), ids=np.array([0]))
try:
    flowpipe.batched_velocity_step(np.zeros((1, 4)), bad, sched)
    raise SystemExit("off-grid t accepted")
except flowpipe.TimeDomainError:
    pass
try:
    flowpipe.batched_velocity_step(np.zeros((2, 4)), bad, sched)
    raise SystemExit("shape mismatch accepted")
except flowpipe.ParameterError:
    pass
print("binding ok", len(cases))
"""


def test_reference_side_ctypes_binding_is_bit_exact():
    if not os.path.isdir(os.path.join(REF, "flowpipe")):
        pytest.skip("reference install baseline/_ref absent (pip install --target baseline/_ref /root/reference)")
    lib = os.path.join(ROOT, "paper_2511_22009_b200", "libstreamflow.so")
    code = f"REF = {REF!r}; ROOT = {ROOT!r}; LIB = {lib!r}\n" + SCRIPT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "binding ok 4" in out.stdout
