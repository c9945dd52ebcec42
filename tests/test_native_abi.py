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
    with pytest.raises(ValueError):
        P.build_problem(inst, object())        # neither FomOperators nor ParameterPoint
    with pytest.raises(ValueError):
        P.init_guess(inst, P.ParameterPoint(100.0, 10.0),
                     ops=P.assemble(inst.grid, P.ParameterPoint(200.0, 10.0)))


def _artifacts(name="tiny_nm"):
    import paper_2305_15163_b200 as P
    from .conftest import golden_path
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    art, keep = inst._artifacts_struct()
    return inst, art, keep


@pytest.mark.parametrize("mutate,msg", [
    (lambda a: setattr(a, "abi_version", 1), "ABI version"),
    (lambda a: setattr(a, "n_blocks", 0), "blocks"),
    (lambda a: setattr(a, "n_blocks", 17), "blocks"),
    (lambda a: setattr(a, "n_c", 0), "multiplier"),
    (lambda a: setattr(a, "nx", 1), "grid"),
    (lambda a: setattr(a, "nu", 0.0), "grid"),
    (lambda a: setattr(a, "map_kind", 7), "map kind"),
    (lambda a: setattr(a, "constraint_mode", 5), "constraint mode"),
    (lambda a: setattr(a.blocks[1], "n_int", a.blocks[0].n_int + 1), "latent dims"),
    (lambda a: setattr(a.blocks[0], "n_cols", a.blocks[0].n_cols + 1), "n_cols"),
    (lambda a: setattr(a.blocks[0], "n_rows", 0), "sample row set is empty"),
    (lambda a: setattr(a.blocks[0], "CA", None), "CA"),
    (lambda a: setattr(a.blocks[0].interior, "n_out", a.blocks[0].interior.n_out + 1),
     "n_io"),
])
def test_ctx_create_rejects_malformed_artifacts(mutate, msg):
    """ddnm_ctx_create validates the artifacts before touching a device
    (ValueError / NotImplementedError as the reference's ValueErrors)."""
    from paper_2305_15163_b200 import _native as N
    inst, art, keep = _artifacts()
    mutate(art)
    h = C.c_void_p()
    rc = N.lib().ddnm_ctx_create(-1, C.byref(art), 0, C.byref(h))
    assert rc in (-1, -3) and not h.value
    assert msg.lower() in N.lib().ddnm_last_error().decode().lower()


def test_gio_out_of_range_rejected():
    from paper_2305_15163_b200 import _native as N
    inst, art, keep = _artifacts()
    blk = art.blocks[0]
    bad = np.ascontiguousarray(np.full(blk.n_gio, 10 ** 9, dtype=np.int64))
    keep.append(bad)
    blk.gio = N.ptr(bad, C.c_int64)
    h = C.c_void_p()
    assert N.lib().ddnm_ctx_create(-1, C.byref(art), 0, C.byref(h)) == -1
    assert "gio" in N.lib().ddnm_last_error().decode()


def test_null_and_range_arguments():
    from paper_2305_15163_b200 import _native as N
    L = N.lib()
    assert L.ddnm_ctx_create(-1, None, 0, None) == -1
    assert L.ddnm_dd_packet_len(None, 0, 1, None) == -1
    assert L.ddnm_binio_read(None, None) == -1
    assert L.ddnm_binio_write(None, 0, None, None, None, None, None) == -1
    assert L.ddnm_ipc_get_handle(None, None) == -1
    n = C.c_int64()
    assert L.ddnm_binio_count(None, C.byref(n)) == -1
