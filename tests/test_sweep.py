"""The device sweep driver (paper_2002_00917_b200.sweep; cli.py:200-266)
against the reference CLI's own sweep output on the same problems
(tests/golden/make_golden_sweep.py -> tests/golden/sweep_cases.json).

Bars: per row the same converged flag and iterations within +-2 (SURVEY §8d rule);
fill_ilu identical to the reference's printed value (the factors are bit-identical) and
equal on every row of an m / rank sweep (one set of ILU factors reused, as
test_cli.py:104-116 asserts); fill_lowrank identical (same achieved rank, same q).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, have_cuda
from oracle import pslr_oracle as O

with open(os.path.join(GOLDEN_DIR, "sweep_cases.json")) as fh:
    SW = json.load(fh)["cases"]


def _params(args):
    """CLI flags of a golden case -> (A, sweep keyword arguments)."""
    kv = dict(zip(args[0::2], args[1::2]))
    nx, ny, nz, shift = kv["--problem"].split(":")[1].split(",")
    A = O.laplacian3d(int(nx), int(ny), int(nz), shift=float(shift))
    kw = {"axis": kv["--axis"], "values": [int(v) for v in kv["--values"].split(",")]}
    for flag, key in (("--s", "s"), ("--m", "m"), ("--rank", "rank"), ("--seed", "seed"),
                      ("--restart", "restart"), ("--maxit", "maxit")):
        if flag in kv:
            kw[key] = int(kv[flag])
    return A, kw


def test_sweep_rejects_bad_axis_and_empty_values():
    import paper_2002_00917_b200 as pg
    A = O.laplacian3d(4, 4, 4, 0.0)
    with pytest.raises(ValueError):
        pg.sweep(A, "q", [1])
    with pytest.raises(ValueError):
        pg.sweep(A, "m", [])


@pytest.mark.gpu
@pytest.mark.skipif(not have_cuda(), reason="needs a CUDA device")
@pytest.mark.parametrize("name", sorted(SW))
def test_device_sweep_matches_reference_cli(name):
    import paper_2002_00917_b200 as pg
    case = SW[name]
    A, kw = _params(case["args"])
    rows, csv = pg.sweep(A, **kw)
    assert csv.splitlines()[0] == ",".join(pg.SWEEP_COLUMNS)
    assert len(rows) == len(case["rows"])
    for got, ref in zip(rows, case["rows"]):
        assert str(got["value"]) == ref["value"]
        assert str(got["converged"]) == ref["converged"]
        assert abs(got["its"] - int(ref["its"])) <= 2, (got["value"], got["its"], ref["its"])
        assert f"{got['fill_ilu']:.6f}" == ref["fill_ilu"]
        assert f"{got['fill_lowrank']:.6f}" == ref["fill_lowrank"]
    if kw["axis"] != "s":
        assert len({r["fill_ilu"] for r in rows}) == 1
    if kw["axis"] == "rank":
        fills = [r["fill_lowrank"] for r in rows]
        assert all(a < b for a, b in zip(fills, fills[1:])) or len(set(fills)) < len(fills)
