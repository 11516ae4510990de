"""CTA-0 clock64 timeline of one layer GEMM (library built with -DSF_GEMM_TRACE=1):
per tile, MMA start (accumulator free) / MMA issue done / epilogue ready / epilogue got accumulator."""
import ctypes, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_22009_b200 import _lib
which = sys.argv[1] if len(sys.argv) > 1 else "fc1"
M, D, T, H = 131072, 384, 1024, 6
st = torch.cuda.current_stream().cuda_stream
bf = lambda t: t.to(torch.bfloat16)
a = bf(torch.randn(M, D, device="cuda"))
h = bf(torch.randn(M, 4 * D, device="cuda"))
if which == "qkv":
    w = bf(torch.randn(3 * D, D, device="cuda") * 0.05); b = torch.zeros(3 * D, device="cuda")
    q = torch.empty(M // T, H, T, 64, device="cuda", dtype=torch.bfloat16); k = torch.empty_like(q)
    vt = torch.empty(M // T, H, 64, T, device="cuda", dtype=torch.float16)
    call = lambda: _lib.call("sf_gemm_qkv", a.data_ptr(), w.data_ptr(), b.data_ptr(), q.data_ptr(), k.data_ptr(),
                             vt.data_ptr(), M, H, T, 0.125, st)
elif which == "fc1":
    w = bf(torch.randn(4 * D, D, device="cuda") * 0.05); b = torch.zeros(4 * D, device="cuda")
    o = torch.empty(M, 4 * D, device="cuda", dtype=torch.bfloat16)
    call = lambda: _lib.call("sf_gemm_bf16", a.data_ptr(), w.data_ptr(), b.data_ptr(), o.data_ptr(), M, 4 * D, D, 2, st)
else:
    A, K = (a, D) if which == "proj" else (h, 4 * D)
    w = bf(torch.randn(D, K, device="cuda") * 0.05); b = torch.zeros(D, device="cuda")
    xres = bf(torch.randn(M, D, device="cuda")); xmod = torch.empty_like(xres)
    vec = torch.randn(M // T, 3 * D, device="cuda") * 0.1
    call = lambda: _lib.call("sf_gemm_res_ln", A.data_ptr(), w.data_ptr(), b.data_ptr(), xres.data_ptr(), xmod.data_ptr(),
                             vec.data_ptr(), vec[:, D:].data_ptr(), vec[:, 2 * D:].data_ptr(), 3 * D, M, D, K, T, 1e-6, st)
for _ in range(3):
    call()
torch.cuda.synchronize()
buf = np.zeros(8 * 64, dtype=np.int64)
lib = ctypes.CDLL(_lib.LIB_PATH)
assert lib.sf_gemm_trace_read(buf.ctypes.data_as(ctypes.c_void_p)) == 0
tr = buf.reshape(8, 64)
t0 = tr[0, 0]
rows = (0, 1, 2, 3)
print("tile  mma_start  mma_issued  epi_ready  epi_got_acc" + "   (cycles; mma_issued = last MMA of the tile issued)")
for i in range(int(os.environ.get('NT', 12))):
    print(f"{i:4d} " + " ".join(f"{(tr[r, i] - t0) if tr[r, i] else -1:11d}" for r in rows))
if which == "qkv":
    print("chunk  acquired  tmem_in_regs  staged  released")
    for i in range(min(63, 3 * int(os.environ.get('NT', 12)))):
        print(f"{i // 3:3d}.{i % 3} " + " ".join(f"{(tr[r, i] - t0) if tr[r, i] else -1:9d}" for r in (4, 5, 6, 7)))
