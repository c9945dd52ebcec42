"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/ddnm.h declares; struct layouts agree; no compute without a GPU."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from .conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ddnm.h")


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ddnm_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2305_15163_b200 import _native as N
    L = N.lib()
    names = header_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(N.EXPORTED)
    assert L.ddnm_abi_version() == N.ABI_VERSION


def test_ctypes_layout_matches_header():
    from paper_2305_15163_b200 import _native as N
    # field order/names of the C structs, parsed from the header
    txt = open(HEADER).read()
    for cname, py in (("ddnm_decoder", N.Decoder), ("ddnm_block", N.Block),
                      ("ddnm_sqp_cfg", N.SqpCfg), ("ddnm_solve_out", N.SolveOut),
                      ("ddnm_eval_out", N.EvalOut), ("ddnm_info", N.Info)):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + cname + ";", txt).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        fields = []
        for decl in body.split(";"):
            decl = decl.strip()
            if not decl:
                continue
            for piece in decl.split(","):
                fields.append(piece.replace("*", " ").split()[-1].split("[")[0])
        assert [f[0] for f in py._fields_] == fields, cname


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2305_15163_b200 as P
    from .conftest import golden_path
    inst = P.RomInstance.load(golden_path("tiny_nm", "artifacts"))
    with pytest.raises(Exception) as ei:
        P.solve_rom_batch(inst, P.seeded_parameters(2))
    assert "CUDA" in str(ei.value) or "device" in str(ei.value)


def test_argument_validation_before_device():
    import paper_2305_15163_b200 as P
    from .conftest import golden_path
    inst = P.RomInstance.load(golden_path("tiny_nm", "artifacts"))
    with pytest.raises(ValueError):
        P.solve_rom_batch(inst, np.zeros((2, 3)))
    with pytest.raises(ValueError):
        P.solve_rom_batch(inst, np.array([[np.nan, 10.0]]))
    with pytest.raises(ValueError):
        P.SqpConfig(backtrack_factor=1.5)
    with pytest.raises(NotImplementedError):
        P.solve_rom(inst, P.ParameterPoint(100.0, 10.0), compute_error=True)
