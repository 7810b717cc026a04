"""The native design reader (model.parse_design_arrays, p3d_parse.cu; SURVEY
8f rank 2) against the reference's parse_design + NetlistArrays on fixtures
the reference produced (tests/golden/parse_cases.json, make_golden.py
--parse): the same arrays (sha256 per field), die / HBT scalars and names for
well-formed text, the same ParseError message for every malformed variant.
Host code: runs on CPU."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2403_09070_b200.model import ParseError, parse_design_arrays

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "parse_cases.json")))


def _digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype}:{a.shape}"


@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_matches_reference(name):
    c = CASES[name]
    if c["error"] is None:
        d = parse_design_arrays(c["text"])
        a = d.arrays()
        for f, want in c["fields"].items():
            assert _digest(getattr(a, f)) == want, f
        die = d.die
        assert [die.width, die.height, die.row_height_top, die.row_height_bottom,
                die.max_util_top, die.max_util_bottom] == c["die"]
        assert [d.hbt.pitch, d.hbt.spacing, d.hbt.cost] == c["hbt"]
        assert d.inst_names == c["inst_names"] and d.net_names == c["net_names"]
    else:
        with pytest.raises(ParseError) as e:
            parse_design_arrays(c["text"])
        assert str(e.value) == c["error"]
