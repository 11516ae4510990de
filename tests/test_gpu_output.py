"""`generate` CSV output, byte-identical to the UNMODIFIED reference's
`flowpipe generate` (fixtures: tests/golden/make_generate_golden.py), i.e. the
reference's acceptance criterion 8 (tests/test_acceptance.py:224-231) against
the reference's own bytes, through the device pipeline."""

import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {
    "n3_s4_seed123": dict(num_images=3, steps=4, seed=123),
    "n4_s4_seed123": dict(num_images=4, steps=4, seed=123),
    "n5_s2_seed7_w7.5": dict(num_images=5, steps=2, seed=7, guidance=7.5),
    "n2_s8_seed0_compiled": dict(num_images=2, steps=8, seed=0, engine="compiled"),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_generate_csv_byte_identical_to_reference(name, tmp_path):
    from paper_2511_22009_b200.output import generate

    want = open(os.path.join(HERE, "golden", "generate", f"{name}.csv"), "rb").read()
    path = tmp_path / "out.csv"
    text = generate(**CASES[name], out=str(path))
    assert path.read_bytes() == want
    assert text.encode() == want


def test_results_csv_format():
    from paper_2511_22009_b200.output import results_csv
    from paper_2511_22009_b200.pipeline import GenerationResult

    r = [GenerationResult(id=1, latent=np.array([0.1, -2.5]), decoded=None, iterations_spanned=2)]
    assert results_csv(r) == "id,dim,values...\n1,2,0.1,-2.5\n"
