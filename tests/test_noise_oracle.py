"""The generation-noise oracle (oracle/noise_oracle.py) pinned against numpy itself:
the reference's generation_noise is np.random.default_rng([seed, id]).standard_normal
(flowpipe src/pipeline.py:92-98), so numpy is the golden source here."""

import math
import random

import numpy as np
import pytest

from oracle import noise_oracle as N

ENTROPIES = [[0, 0], [1, 0], [42, 7], [2**32 - 1, 2**32], [2**40 + 3, 2**33 + 1], [123456789, 2**62]]


@pytest.mark.parametrize("vals", ENTROPIES)
def test_seed_sequence_and_pcg64_state(vals):
    want = [int(v) for v in np.random.SeedSequence(vals).generate_state(4, np.uint64)]
    assert N.seed_sequence_state(vals, 4) == want
    bg = np.random.PCG64(np.random.SeedSequence(vals))
    p = N.PCG64(vals)
    assert (p.state, p.inc) == (bg.state["state"]["state"], bg.state["state"]["inc"])
    assert [p.next64() for _ in range(8)] == [int(v) for v in bg.random_raw(8)]


@pytest.mark.parametrize("seed,gen", [(0, 0), (42, 7), (2**40 + 3, 2**33 + 1)])
def test_standard_normal_bit_exact(seed, gen):
    want = np.random.default_rng([seed, gen]).standard_normal(20000)
    got = N.generation_noise(seed, gen, 20000)
    assert np.array_equal(want.view(np.uint64), got.view(np.uint64))


def test_sample_reaches_tail_and_wedge():
    """The 20000-draw samples above exercise the idx==0 tail (|x| > r) and wedge paths."""
    x = np.concatenate([np.random.default_rng([s, 1]).standard_normal(20000) for s in range(3)])
    assert (np.abs(x) > N.ZIG_R).sum() >= 3


def test_tables_match_numpy_header_values():
    ki, wi, fi = N.load_tables()
    assert ki[0] == 0x000EF33D8025EF6A and ki[1] == 0 and fi[0] == 1.0
    assert wi[0] == 8.68362706080130616677e-16
    assert all(fi[i] > fi[i + 1] for i in range(255)) and len(ki) == len(wi) == len(fi) == 256


def test_glibc_log1p_restatement_bit_exact():
    """The restated libm log1p (mirrored by csrc/numpy_noise.cu glibc_log1p) equals
    math.log1p (== npy_log1p) on the inputs the ziggurat tail feeds it: -u, u = k/2^53."""
    rng = random.Random(5)
    xs = [-(rng.getrandbits(53) * 2.0**-53) for _ in range(20000)]
    xs += [-(rng.getrandbits(53) * 2.0**-53) * 2.0 ** -rng.randint(0, 60) for _ in range(10000)]
    xs += [0.0, -0.0, -2.0**-53, -0.5, -0.2929, -0.29289, -(1 - 2.0**-53), 0.25, 1.5, 1e10]
    bad = [x for x in xs if struct_bits(N.glibc_log1p(x)) != struct_bits(math.log1p(x))]
    assert not bad, bad[:5]


def struct_bits(v: float) -> int:
    return int(np.float64(v).view(np.uint64))
