"""Measured error of the bf16 device DiT against the fp32 oracle (run on the GPU, TF32 off), at
the bench's row count, for the record (profiles/r02s3/numerics.md): per-row normalised max / mean
|eps_dev - eps_fp32| / max|eps_fp32| for DiT-S/2 (128 rows in 8-row oracle chunks) and DiT-XL/2
(8 rows), with the test bounds beside them."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_22009_b200 as sf  # noqa: E402
from oracle.dit_oracle import dit_forward, params_to  # noqa: E402
from paper_2511_22009_b200.dit import DIT_S2, DIT_XL2  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def report(cfg, rows, heads, chunk):
    model = sf.DiTVelocityModel(cfg, seed=9, max_rows=rows, bias_std=0.02)
    dit = model.device_model
    g = torch.Generator().manual_seed(rows)
    x = torch.randn(rows, 4, 64, 64, generator=g).cuda()
    t = torch.rand(rows, generator=g, dtype=torch.float64).cuda()
    e = torch.randn(rows, 8, generator=g, dtype=torch.float64).cuda()
    got = dit.forward(x, t, e).clone()
    pg = params_to(model.params, "cuda")
    mx, mean = [], []
    for r in range(0, rows, chunk):
        want = dit_forward(pg, x[r:r + chunk], t[r:r + chunk], e[r:r + chunk], heads=heads).reshape(chunk, -1)
        err = (got[r:r + chunk] - want).abs()
        scale = want.abs().amax(dim=1)
        mx += (err.amax(dim=1) / scale).tolist()
        mean += (err.mean(dim=1) / scale).tolist()
    mx, mean = np.array(mx), np.array(mean)
    return (f"| {cfg.name if hasattr(cfg, 'name') else cfg.hidden} | {rows} | {np.median(mx):.2e} | {mx.max():.2e} | "
            f"{np.median(mean):.2e} | {mean.max():.2e} |")


print("| model (hidden) | rows | max err, median row | max err, worst row | mean err, median row | mean err, worst row |")
print("|---|---|---|---|---|---|")
print(report(DIT_S2, 128, 6, 8))
print(report(DIT_XL2, 8, 16, 2))
