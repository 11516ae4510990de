"""clock64 timeline of the pair block tail (cluster 0) at the bench shape.

    python tools/tail_trace.py            (builds build_trace/libstreamflow_trace.so with -DSF_TAIL2_TRACE=1)

Rows per CTA: MMA (leader) tile marks [a2empty wait, a2empty ok, xready ok, MLP done],
worker tile marks [proj epi start, xready arrive, final epi start, xfree], per-chunk
[GELU a1full ok], [MMA before a1empty], [after], [before hfull], [after], [GELU before hempty]."""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "build_trace", "libstreamflow_trace.so")


def build():
    from paper_2511_22009_b200 import build as B

    os.makedirs(os.path.join(ROOT, "build_trace"), exist_ok=True)
    objs = []
    for src in B._sources():
        obj = os.path.join(ROOT, "build_trace", os.path.basename(src).replace(".cu", ".o"))
        subprocess.run([B.NVCC, *B.FLAGS, "-DSF_TAIL2_TRACE=1", "-c", src, "-o", obj], check=True)
        objs.append(obj)
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "shared", "-o", LIB, *objs,
                    "-Xlinker", "-rpath=/usr/local/cuda/lib64"], check=True)


if __name__ == "__main__":
    if not os.path.exists(LIB) or "--build" in sys.argv:
        build()
        if "--build-only" in sys.argv:
            sys.exit(0)
    os.environ["SF_LIB_PATH"] = LIB
    import torch

    from paper_2511_22009_b200 import _lib

    T, N, F = 1024, 384, 1536
    slots = int(os.environ.get("SLOTS", "128"))
    M = slots * T
    g = torch.Generator(device="cuda").manual_seed(0)
    bf = lambda x: x.to(torch.bfloat16)
    attn = bf(torch.randn(M, N, device="cuda", generator=g))
    wp = bf(torch.randn(N, N, device="cuda", generator=g) * 0.05)
    w1 = bf(torch.randn(F, N, device="cuda", generator=g) * 0.05)
    w2 = bf(torch.randn(N, F, device="cuda", generator=g) * 0.03)
    bp, b1, b2 = (torch.zeros(n, device="cuda") for n in (N, F, N))
    xres = bf(torch.randn(M, N, device="cuda", generator=g))
    xmod = torch.empty_like(xres)
    vecs = torch.randn(slots, 8 * N, device="cuda", generator=g) * 0.1
    P = lambda t: t.data_ptr()
    st = torch.cuda.current_stream().cuda_stream
    args = [P(attn), P(wp), P(bp), P(w1), P(w2), P(b1), P(b2), P(xres), P(xmod)] + \
           [P(vecs[:, i * N:]) for i in range(6)] + [8 * N, 1e-6, M, T, st]
    for _ in range(3):
        _lib.call("sf_block_tail", *args)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        _lib.call("sf_block_tail", *args)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"block tail: {ev[0].elapsed_time(ev[1]) / 10 * 1e3:.1f} us per launch at M={M}")
    buf = np.zeros(16 * 128, dtype=np.int64)
    assert ctypes.CDLL(LIB).sf_tail2_trace_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
    tr = buf.reshape(16, 128)
    t0 = tr[:, :64][tr[:, :64] > 0].min()
    rel = lambda r, i: int(tr[r, i] - t0) if tr[r, i] else -1
    print("epilogue marks (CTA 0, worker e0): [acc ok, rows ok, res pass done, x stored, LN done, (final) xmod stored]")
    for t in range(2):
        for k, nm in ((0, "proj "), (8, "final")):
            print(t, nm, [int(tr[1, 32 + 16 * t + k + i] - t0) if tr[1, 32 + 16 * t + k + i] else -1 for i in range(6)])
    print("MMA warp cumulative wait cycles per tile end: wfull, a1empty, hfull")
    for t in range(7):
        print(t, tr[0, 64 + 4 * t], tr[0, 64 + 4 * t + 1], tr[0, 64 + 4 * t + 2])
    for cta in (0, 1):
        base = 8 * cta
        print(f"--- CTA {cta}")
        print("tile  mma:a2e-wait  a2e-ok  xready-ok  mlp-done | wk:proj-epi  xready-arr  final-epi  xfree")
        for t in range(8):
            print(f"{t:3d} " + " ".join(f"{rel(base + 0, 4 * t + k):10d}" for k in range(4)) + " | " +
                  " ".join(f"{rel(base + 1, 4 * t + k):10d}" for k in range(4)))
        print("chunk  gelu-a1full  mma:pre-a1e  a1e-ok  pre-hfull  hfull-ok  gelu:pre-hempty  gelu:ld-done  gelu:arrived")
        for c in range(40):
            print(f"{c:3d} " + " ".join(f"{rel(base + r, c):10d}" for r in (2, 3, 4, 5, 6, 7)) +
                  (f" {int(tr[base + 1, 64 + c] - t0):10d} {int(tr[base + 1, 96 + c] - t0):10d}" if c < 32 else ""))
