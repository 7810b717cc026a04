"""The fast array generator reproduces place3d.synth.gen_synthetic ->
parse_design -> NetlistArrays exactly (golden sha256 digests from the reference)."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2403_09070_b200.synth import SynthSpec, synth_arrays

GOLD = os.path.join(os.path.dirname(__file__), "golden", "synth_checksums.json")
CHECKS = json.load(open(GOLD))


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype}:{a.shape}"


@pytest.mark.parametrize("name", ["tiny", "small", "cfg1", "cfg2"])
def test_arrays_match_reference(name):
    ref = CHECKS[name]
    d = synth_arrays(SynthSpec(**ref["spec"]))
    a = d.arrays()
    for f, want in ref["fields"].items():
        assert digest(getattr(a, f)) == want, f
    die = d.die
    assert [die.width, die.height, die.row_height_top, die.row_height_bottom,
            die.max_util_top, die.max_util_bottom] == ref["die"]
    assert [d.hbt.pitch, d.hbt.spacing, d.hbt.cost] == ref["hbt"]


def test_cache_roundtrip(tmp_path):
    from paper_2403_09070_b200.synth import cached_synth

    spec = SynthSpec(**CHECKS["tiny"]["spec"])
    a = cached_synth(spec, cache_dir=str(tmp_path)).arrays()
    b = cached_synth(spec, cache_dir=str(tmp_path)).arrays()
    for f in CHECKS["tiny"]["fields"]:
        assert np.array_equal(getattr(a, f), getattr(b, f))
