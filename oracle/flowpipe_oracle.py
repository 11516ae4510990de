"""CPU oracle for the StreamFlow stream-batch hot path (TEST INFRASTRUCTURE ONLY).

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product package
(``paper_2511_22009_b200``) never imports anything under ``oracle/``.

It restates, in plain numpy, the reference package ``flowpipe``
(``/root/reference/pkg/src/flowpipe``) for every function on the hot path:

* noise table / window schedule      -> ``schedule.py:63-173``
* per-timestep window coefficients    -> ``schedule.py:201-263``
* grid successor                      -> ``schedule.py:266-295``
* heterogeneous-t Euler step          -> ``velocity.py:93-135``
* seeded mock velocity model          -> ``models.py:188-241``
* classifier-free guidance            -> ``models.py:244-296``
* generation noise sub-seeding        -> ``pipeline.py:92-98``
* the stream batch (Alg. 2)           -> ``pipeline.py:139-220``

Parity pin: every function here is checked against the reference's own
golden vectors (``tests/test_*.py`` constants) and
against fixtures produced by importing the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/flowpipe_golden.npz``); see
``tests/test_oracle_golden.py``.  Arithmetic is written in the same literal
operation order as the reference, so agreement is bit-for-bit.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# schedule (reference schedule.py:25-30 defaults, :63-84 noise table)
# ---------------------------------------------------------------------------

T_MAX = 1000
BETA_START = 1e-4
BETA_END = 0.02
NUM_WINDOWS = 4
EPS = 1e-6


@dataclass(frozen=True)
class OracleSchedule:
    """Window partition + noise table + inference grid (schedule.py:87-133)."""

    boundaries: np.ndarray  # [K+1] fp64
    abar: np.ndarray  # [t_max] fp64
    grid: np.ndarray  # [n] fp64
    eps: float = EPS

    @property
    def t_max(self) -> int:
        return len(self.abar)


def noise_table(t_max: int = T_MAX, beta_start: float = BETA_START,
                beta_end: float = BETA_END) -> np.ndarray:
    """alpha-bar = cumprod(1 - linspace(beta_start, beta_end)) (schedule.py:79-81)."""
    betas = np.linspace(beta_start, beta_end, t_max, dtype=np.float64)
    return np.cumprod(1.0 - betas)


def make_schedule(num_windows: int = NUM_WINDOWS, steps: int = 4,
                  boundaries=None, grid=None, abar=None, eps: float = EPS) -> OracleSchedule:
    """Equal windows via linspace (schedule.py:162), grid i/n (schedule.py:136-140)."""
    if boundaries is None:
        boundaries = np.linspace(0.0, 1.0, num_windows + 1, dtype=np.float64)
    if grid is None:
        grid = np.arange(steps, dtype=np.float64) / float(steps)
    if abar is None:
        abar = noise_table()
    return OracleSchedule(np.asarray(boundaries, np.float64), np.asarray(abar, np.float64),
                          np.asarray(grid, np.float64), float(eps))


def _abar_at(tau: float, sch: OracleSchedule) -> float:
    """Round-half-up table index of flow time tau, clamped (schedule.py:201-205)."""
    raw = (1.0 - tau) * float(sch.t_max - 1)
    idx = int(np.floor(raw + 0.5))
    idx = min(max(idx, 0), sch.t_max - 1)
    return float(sch.abar[idx])


def window_of(t: float, sch: OracleSchedule) -> int:
    """Masked count of interior boundaries below t (+eps), ties -> lower window
    (schedule.py:208-221)."""
    if not (0.0 <= t <= 1.0):
        raise ValueError(f"TimeDomainError: t={t} outside [0, 1]")
    inner = sch.boundaries[1:-1]
    return int(np.count_nonzero(t > inner + sch.eps))


def grid_successor(t: float, sch: OracleSchedule) -> float:
    """Nearest grid point within eps, then its successor in grid + [1.0]
    (schedule.py:266-295)."""
    if not (0.0 <= t <= 1.0):
        raise ValueError(f"TimeDomainError: t={t} outside [0, 1]")
    g = sch.grid
    pos = int(np.searchsorted(g, t))
    lo = min(max(pos - 1, 0), len(g) - 1)
    hi = min(max(pos, 0), len(g) - 1)
    idx = hi if abs(g[hi] - t) <= abs(g[lo] - t) else lo
    if abs(g[idx] - t) > sch.eps:
        raise ValueError(f"TimeDomainError: t={t} not on the inference grid")
    return 1.0 if idx + 1 == len(g) else float(g[idx + 1])


@dataclass(frozen=True)
class StepCoeffs:
    """Everything the Euler step needs for one flow time (schedule.py:224-263,
    velocity.py:115-129), all fp64."""

    t: float
    t_next: float
    t_s: float
    t_e: float
    gamma: float
    lambda_s: float
    eta_s: float
    lambda_t: float
    eta_t: float
    span: float
    dt: float
    at_end: bool


def window_coeffs(t: float, sch: OracleSchedule) -> tuple:
    """(t_s, t_e, gamma, lambda_s, eta_s, lambda_t, eta_t) of one flow time,
    literal reference operation order (schedule.py:238-262)."""
    k = window_of(t, sch)
    t_s = float(sch.boundaries[k])
    t_e = float(sch.boundaries[k + 1])
    gamma = float(np.sqrt(_abar_at(t_s, sch) / _abar_at(t_e, sch)))
    lambda_s = 1.0 / gamma
    eta_s = -float(np.sqrt(1.0 - gamma * gamma)) / gamma
    denom = lambda_s * (t - t_s) + (t_e - t)
    if denom <= 0.0:
        raise ArithmeticError("InvariantError: non-positive window denominator")
    lambda_t = lambda_s * (t_e - t_s) / denom
    eta_t = eta_s * (t_e - t) / denom
    return t_s, t_e, gamma, lambda_s, eta_s, lambda_t, eta_t


def step_coeffs(t: float, sch: OracleSchedule) -> StepCoeffs:
    """Window coefficients plus grid successor of one on-grid timestep
    (schedule.py:224-295; velocity.py:115-129)."""
    t_s, t_e, gamma, lambda_s, eta_s, lambda_t, eta_t = window_coeffs(t, sch)
    t_next = grid_successor(t, sch)
    span = t_e - t
    return StepCoeffs(t, t_next, t_s, t_e, gamma, lambda_s, eta_s, lambda_t, eta_t,
                      span, t_next - t, span <= sch.eps)


def euler_step(eps_hat: np.ndarray, x: np.ndarray, ts, sch: OracleSchedule) -> tuple[np.ndarray, np.ndarray]:
    """Heterogeneous-t Euler update of a [B, D] block (velocity.py:93-135).

    Coefficients are fp64 and cast to the latent dtype before the three
    elementwise passes; at-window-end rows keep v = 0 exactly.
    """
    x = np.asarray(x)
    dt_ = x.dtype
    out = np.empty_like(x)
    t_next = np.empty(len(ts), np.float64)
    for i, t in enumerate(np.asarray(ts, np.float64)):
        c = step_coeffs(float(t), sch)
        t_next[i] = c.t_next
        xi = x[i]
        e = np.asarray(eps_hat[i]).astype(dt_, copy=False)
        x_pred = dt_.type(c.lambda_t) * xi + dt_.type(c.eta_t) * e
        if c.at_end:
            v = np.zeros_like(xi)
        else:
            v = (x_pred - xi) / dt_.type(c.span)
        out[i] = xi + dt_.type(c.dt) * v
    return out, t_next


# ---------------------------------------------------------------------------
# seeded mock velocity model (models.py:188-241)
# ---------------------------------------------------------------------------

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mock_row_key(model_seed: int, gen_id: int, t: float, emb: np.ndarray) -> int:
    """blake2b-64 over <qqq(seed, id, round(t*1e9)) || emb fp64 bytes (models.py:223-228)."""
    msg = struct.pack("<qqq", int(model_seed), int(gen_id), int(round(float(t) * 1e9)))
    msg += np.ascontiguousarray(emb, dtype="<f8").tobytes()
    return int.from_bytes(hashlib.blake2b(msg, digest_size=8).digest(), "little")


def splitmix_expand(key: int, dim: int) -> np.ndarray:
    """splitmix64 finaliser per coordinate, mapped to [-1, 1) (models.py:188-196)."""
    with np.errstate(over="ignore"):
        z = np.uint64(key) ^ (np.arange(dim, dtype=np.uint64) * _GOLD)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


def mock_eps(model_seed: int, ids, ts, row_embs, dim: int) -> np.ndarray:
    """Mock forward for a batch: row i = f(seed, id_i, t_i, emb_i) (models.py:230-236)."""
    return np.stack([splitmix_expand(mock_row_key(model_seed, g, t, e), dim)
                     for g, t, e in zip(ids, ts, row_embs)], axis=0)


def guided_mock_eps(model_seed: int, ids, ts, emb, neg, w: float, dim: int) -> np.ndarray:
    """apply_cfg -> forward -> handle_cfg (models.py:244-296, pipeline.py:109-121)."""
    b = len(ids)
    if w == 1.0:
        return mock_eps(model_seed, ids, ts, [emb] * b, dim)
    neg = np.zeros_like(emb) if neg is None else neg
    eu = mock_eps(model_seed, ids, ts, [neg] * b, dim)
    ec = mock_eps(model_seed, ids, ts, [emb] * b, dim)
    return eu + w * (ec - eu)


# ---------------------------------------------------------------------------
# stream batch (pipeline.py:92-98, :139-220)
# ---------------------------------------------------------------------------


def generation_noise(seed: int, gen_id: int, dim: int) -> np.ndarray:
    """PCG64 sub-seeded by [seed, id], standard normal (pipeline.py:92-98)."""
    return np.random.default_rng([seed, gen_id]).standard_normal(dim)


def conditioning_embedding(seed: int, embed_dim: int = 8) -> np.ndarray:
    """Seed-derived conditioning vector (config.py:284-289)."""
    return np.random.default_rng([seed, 2 ** 32 - 1]).standard_normal(embed_dim)


@dataclass
class OracleRun:
    latents: dict  # gen id -> final latent
    order: list  # completion order of gen ids
    spans: dict  # gen id -> iterations spanned
    batch_ids: list  # per iteration: ids in batch order (newest first)
    batch_ts: list  # per iteration: timesteps in batch order
    model_calls: int = 0
    scheduler_calls: int = 0
    param_evals: int = 0
    decodes: int = 0
    snapshots: list = field(default_factory=list)


def run_stream(m: int, n: int, eps_fn, seed: int, sch: OracleSchedule, dim: int,
               dtype=np.float64, keep_snapshots: bool = False) -> OracleRun:
    """Alg. 2 written against the closed-form queue of SURVEY Appendix A:
    at iteration j the batch holds generations hi..lo (newest first) with
    lo = max(0, j-n+1), hi = min(j, m-1); generation g is at stage j-g.
    ``eps_fn(ids, ts, x) -> [B, D]`` is the (guided) velocity model.
    Mirrors pipeline.py:164-220 step for step."""
    state: dict[int, np.ndarray] = {}
    run = OracleRun({}, [], {}, [], [])
    for j in range(m + n - 1):
        if j < m:
            state[j] = generation_noise(seed, j, dim).astype(dtype, copy=False)
        lo, hi = max(0, j - n + 1), min(j, m - 1)
        gens = list(range(hi, lo - 1, -1))
        ts = sch.grid[[j - g for g in gens]]
        x = np.stack([state[g] for g in gens], axis=0)
        eps = eps_fn(np.asarray(gens, np.int64), ts, x)
        x_new, _ = euler_step(eps, x, ts, sch)
        run.model_calls += 1
        run.scheduler_calls += 1
        run.param_evals += len(gens)
        run.batch_ids.append(gens)
        run.batch_ts.append(ts.tolist())
        for i, g in enumerate(gens):
            state[g] = x_new[i]
        if j - lo + 1 == n and lo <= hi:  # oldest entry reached stage n
            run.latents[lo] = state.pop(lo)
            run.order.append(lo)
            run.spans[lo] = j - lo + 1
            run.decodes += 1
        if keep_snapshots:
            run.snapshots.append([(g, j - g + 1, state[g].copy()) for g in gens if g in state])
    return run
