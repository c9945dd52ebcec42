"""Host logic of the evaluation units (csrc/ddnm_abi.cu split_block), on the
CPU through ddnm_plan_units: every sampled row lands in exactly one row unit
of its block, the per-unit limits hold, the constraint units cover the
interface decoder's outputs exactly once, and the accumulate flags mark every
unit but the first of each kind."""

import ctypes as C
import os

import numpy as np
import pytest

import paper_2305_15163_b200 as P
from paper_2305_15163_b200 import _native as N

from .conftest import golden_path

UF_ROWS, UF_CON, UF_ACC_GRAM, UF_ACC_CON = 1, 2, 4, 8


def _plan(name):
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    art, keep = inst._artifacts_struct()
    n = C.c_int32()
    N.check(N.lib().ddnm_plan_units(C.byref(art), C.byref(n), None, None))
    total_rows = sum(int(inst.arrays[f"b{b}_res_rows"].size) for b in range(inst.n_blocks))
    rows = np.full(total_rows, -1, np.int32)
    info = np.zeros((max(n.value, 1), 8), np.int32)
    N.check(N.lib().ddnm_plan_units(C.byref(art), C.byref(n), N.ptr(rows, C.c_int32),
                                    N.ptr(info, C.c_int32)))
    del keep
    return inst, n.value, rows, info[:n.value]


@pytest.mark.parametrize("name", ["c3_nm", "c4_nm"])
def test_large_blocks_split_with_full_coverage(name):
    inst, n, rows, info = _plan(name)
    assert n > inst.n_blocks
    assert np.all(rows >= 0)                                  # every row in a unit
    off = 0
    for b in range(inst.n_blocks):
        nr = int(inst.arrays[f"b{b}_res_rows"].size)
        units = info[:, 0] == b
        ru = np.flatnonzero(units & ((info[:, 1] & UF_ROWS) != 0))
        cu = np.flatnonzero(units & ((info[:, 1] & UF_CON) != 0))
        # rows of block b only in block b's row units, counts add up
        assert set(np.unique(rows[off:off + nr])) == set(ru.tolist())
        assert info[ru, 2].sum() == nr
        assert np.all(info[ru, 2] <= 128)                    # row limit
        # hidden-unit limit (a single row may exceed it on its own)
        assert np.all((info[ru, 4] <= 1536) | (info[ru, 2] == 1))
        # constraint units partition the interface outputs; their C A_i columns match
        ngo = int(inst.arrays[f"b{b}_gam_W1"].shape[0]) and int(inst.arrays[f"b{b}_n_interface"])
        assert info[cu, 5].sum() == ngo and np.array_equal(info[cu, 5], info[cu, 7])
        # first unit of each kind writes, the others accumulate
        assert (info[ru[0], 1] & UF_ACC_GRAM) == 0 and np.all(info[ru[1:], 1] & UF_ACC_GRAM)
        assert (info[cu[0], 1] & UF_ACC_CON) == 0 and np.all(info[cu[1:], 1] & UF_ACC_CON)
        off += nr


def test_small_blocks_stay_whole_unless_forced(monkeypatch):
    _, n, _, _ = _plan("c0_nm")
    assert n == 0
    monkeypatch.setenv("DDNM_UNIT_ROWS", "24")
    inst, n, rows, info = _plan("c0_nm")
    assert n > inst.n_blocks and np.all(rows >= 0)
    assert np.all(info[(info[:, 1] & UF_ROWS) != 0, 2] <= 24)
