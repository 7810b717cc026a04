"""libp3d.so from plain C (tests/c_consumer/p3d_consumer.c, built here with
gcc against include/p3d.h): the header's structs have the library's sizes and
ABI version, and the native design reader called through the C-ABI reads the
reference-produced parse fixtures exactly as the Python mirror does (which
test_parse.py pins to the reference's parse_design).  Host code: runs on CPU."""

import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from paper_2403_09070_b200.model import ParseError, parse_design_arrays

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2403_09070_b200")
CASES = json.load(open(os.path.join(ROOT, "tests", "golden", "parse_cases.json")))


@pytest.fixture(scope="module")
def consumer(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    if not os.path.exists(os.path.join(LIBDIR, "libp3d.so")):
        from paper_2403_09070_b200 import build

        build.build()
    exe = str(tmp_path_factory.mktemp("c") / "p3d_consumer")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c_consumer", "p3d_consumer.c"), "-L", LIBDIR,
                    "-lp3d", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_abi_and_struct_sizes(consumer):
    out = subprocess.run([consumer], capture_output=True, text=True, check=True).stdout
    assert json.loads(out) == {"abi": 1}


@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_through_c_abi(consumer, tmp_path, name):
    text = CASES[name]["text"]
    path = tmp_path / "design.txt"
    path.write_text(text)
    got = json.loads(subprocess.run([consumer, str(path)], capture_output=True, text=True,
                                    check=True).stdout)
    if CASES[name]["error"] is not None:
        assert got["rc"] == 1 and got["error"] == CASES[name]["error"]
        with pytest.raises(ParseError):
            parse_design_arrays(text)
        return
    d = parse_design_arrays(text)
    a = d.arrays()
    assert got["rc"] == 0
    assert (got["n_inst"], got["n_net"], got["n_pin"]) == (a.n_inst, a.n_net, a.n_pin)
    assert got["n_macro"] == int(a.is_macro.sum())
    assert got["sum_ptr"] == int(a.net_ptr.sum())
    assert got["sum_pin"] == int((a.pin_inst * (np.arange(a.n_pin) % 7 + 1)).sum())
    assert got["sum_size"] == pytest.approx(float((a.w_top + 2 * a.h_top + 3 * a.w_bot
                                                   + 4 * a.h_bot).sum()), rel=1e-15)
    off = a.ox_top + 2 * a.oy_top + 3 * a.ox_bot + 4 * a.oy_bot
    assert got["sum_off"] == pytest.approx(float(off.sum()), rel=1e-12, abs=1e-9)
    die, hbt = d.die, d.hbt
    assert got["scalars"] == [die.width, die.height, die.row_height_top, die.row_height_bottom,
                              die.max_util_top, die.max_util_bottom, hbt.pitch, hbt.spacing,
                              hbt.cost]
