"""binio: the C++ reader/writer in libddnm.so against files
written by the reference itself (tests/golden/ref_*; tools/make_binio_fixtures.py),
the reference's serialized nets, instance files, and a GPU context created
from an instance file by the C entry point alone."""

import os

import numpy as np
import pytest

from .conftest import golden_path, GOLDEN


def _fx(name):
    return os.path.join(GOLDEN, name)


def test_reads_reference_written_matrices_bit_exactly():
    from paper_2305_15163_b200 import binio
    got = binio.read_matrices(_fx("ref_binio_matrices.bin"))
    exp = np.load(_fx("ref_binio_matrices.npz"))
    names = [str(n) for n in exp["names"]]
    assert list(got) == names                       # record order kept
    for i, n in enumerate(names):
        e = exp[f"m{i}"]
        e = e[:, None] if e.ndim == 1 else e        # 1-D arrays are stored as one column
        assert got[n].shape == e.shape and got[n].dtype == np.float64
        # bit patterns (signed zero, nan, subnormal included)
        np.testing.assert_array_equal(got[n].view(np.uint64), np.ascontiguousarray(e).view(np.uint64))


def test_writer_is_byte_identical_to_the_reference(tmp_path):
    from paper_2305_15163_b200 import binio
    exp = np.load(_fx("ref_binio_matrices.npz"))
    names = [str(n) for n in exp["names"]]
    out = tmp_path / "w.bin"
    binio.write_matrices(out, [(n, exp[f"m{i}"]) for i, n in enumerate(names)])
    assert out.read_bytes() == open(_fx("ref_binio_matrices.bin"), "rb").read()


def test_format_errors(tmp_path):
    from paper_2305_15163_b200 import binio
    from paper_2305_15163_b200.errors import FormatError
    raw = open(_fx("ref_binio_matrices.bin"), "rb").read()
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOTMAGIC" + raw[8:])
    with pytest.raises(FormatError, match="bad magic"):
        binio.read_matrices(bad)
    bad.write_bytes(raw[:-3])                        # truncated last record
    with pytest.raises(FormatError, match="overruns|truncated"):
        binio.read_matrices(bad)
    bad.write_bytes(raw[:10])                        # truncated header
    with pytest.raises(FormatError, match="truncated"):
        binio.read_matrices(bad)
    # a record claiming 2^62 x 4 values must not overflow the size check
    hdr = b"DDNMROM1" + (1).to_bytes(4, "little") + b"x" + (1 << 62).to_bytes(8, "little") \
        + (4).to_bytes(8, "little")
    bad.write_bytes(hdr + b"\0" * 64)
    with pytest.raises(FormatError, match="overruns"):
        binio.read_matrices(bad)
    empty = tmp_path / "e.bin"
    empty.write_bytes(b"DDNMROM1")
    assert binio.read_matrices(empty) == {}
    meta = tmp_path / "m.txt"
    meta.write_text("a = 1\nbroken line\n")
    with pytest.raises(FormatError, match="expected 'key = value'"):
        binio.read_meta(meta)


def test_loads_reference_serialized_net():
    """save_net (autoencoder.py:424-450) of the tiny instance's interior net 0
    is exactly that block's full decoder in the artifacts."""
    from paper_2305_15163_b200 import binio
    net = binio.load_net(_fx("ref_net_int0.bin"))
    a = np.load(golden_path("tiny_nm", "artifacts"))
    for k in ("W1", "b1", "W2_indptr", "W2_indices", "W2_data", "scale", "shift"):
        np.testing.assert_array_equal(net[k], a[f"b0_intf_{k}"], err_msg=k)
    assert net["activation"] == "swish" and net["band"] == 4 and net["shift_mask"] == 1
    assert net["W1"].shape == (net["width"], net["latent_dim"])


@pytest.mark.parametrize("name", ["tiny_nm", "c0_ls", "tiny_srpc", "c0_nmg"])
def test_instance_file_round_trip(tmp_path, name):
    import paper_2305_15163_b200 as P
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    path = tmp_path / f"{name}.bin"
    inst.save_binio(path)
    back = P.RomInstance.load(str(path))
    assert back.meta == inst.meta
    assert set(back.arrays) == set(inst.arrays)
    for k, v in inst.arrays.items():
        if k == "meta_json":
            continue
        assert back.arrays[k].shape == v.shape, k
        assert back.arrays[k].dtype == v.dtype, k
        np.testing.assert_array_equal(back.arrays[k], v, err_msg=k)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c0_nm", "c0_srpc", "tiny_ls"])
def test_context_from_instance_file_solves_identically(tmp_path, name):
    """ddnm_ctx_create_binio (no Python in the loop) gives a context whose
    solves and decodes are bitwise those of the npz-built context."""
    import ctypes as C

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200 import _native as N
    from paper_2305_15163_b200.driver import _cfg_struct
    inst = P.RomInstance.load(golden_path(name, "artifacts"))
    path = tmp_path / f"{name}.bin"
    inst.save_binio(path)
    mu = P.seeded_parameters(32, seed=12)
    ref = P.solve_rom_batch(inst, mu)
    L = N.lib()
    h = C.c_void_p()
    N.check(L.ddnm_ctx_create_binio(-1, str(path).encode(), 0, C.byref(h)))
    try:
        B, nD, nC = mu.shape[0], inst.n_primal, inst.n_mult
        x, lam = np.empty((B, nD)), np.empty((B, nC))
        n_iter, status = np.empty(B, np.int32), np.empty(B, np.int32)
        so = N.SolveOut()
        so.x, so.lam = N.ptr(x), N.ptr(lam)
        so.n_iter, so.status = N.ptr(n_iter, C.c_int32), N.ptr(status, C.c_int32)
        N.check(L.ddnm_solve_batch(h, B, N.ptr(np.ascontiguousarray(mu)), None, None,
                                   C.byref(_cfg_struct(P.SqpConfig())), C.byref(so)))
        np.testing.assert_array_equal(x, ref.x)
        np.testing.assert_array_equal(lam, ref.lam)
        np.testing.assert_array_equal(n_iter, ref.n_iter)
        np.testing.assert_array_equal(status, ref.status)
        if inst.has_full_decoders:
            n = C.c_int64()
            N.check(L.ddnm_ctx_state_len(h, C.byref(n)))
            st = np.empty((B, n.value))
            N.check(L.ddnm_decode_batch(h, B, N.ptr(x), None, N.ptr(st), None))
            np.testing.assert_array_equal(st, P.decode_batch(inst, ref.x).states)
    finally:
        L.ddnm_ctx_destroy(h)


@pytest.mark.gpu
def test_c_program_solves_from_instance_file(tmp_path):
    """examples/solve_binio.c: a C caller with no Python (context from an
    instance file, batched solve, binio output) agrees bitwise with the
    Python API on the same parameters."""
    import subprocess

    import paper_2305_15163_b200 as P
    from paper_2305_15163_b200 import binio
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "solve_binio"
    subprocess.run(["gcc", "-O2", "-I", os.path.join(root, "include"),
                    os.path.join(root, "examples", "solve_binio.c"),
                    "-L", os.path.join(root, "paper_2305_15163_b200"), "-lddnm",
                    "-Wl,-rpath," + os.path.join(root, "paper_2305_15163_b200"),
                    "-o", str(exe)], check=True)
    inst = P.RomInstance.load(golden_path("c0_nm", "artifacts"))
    inst.save_binio(tmp_path / "c0.bin")
    out = subprocess.run([str(exe), str(tmp_path / "c0.bin"), "48", str(tmp_path / "out.bin")],
                         check=True, capture_output=True, text=True)
    assert "solved 48 parameters" in out.stdout
    m = binio.read_matrices(tmp_path / "out.bin")
    mu = np.ascontiguousarray(m["mu"].T)
    ref = P.solve_rom_batch(inst, mu)
    np.testing.assert_array_equal(m["latent"].T, ref.x)
    np.testing.assert_array_equal(m["multipliers"].T, ref.lam)


def test_round_trip_property(tmp_path):
    """Random record sets: the C++ writer and reader are inverse, bit for bit
    (names in UTF-8, empty and one-column matrices, any float64 pattern)."""
    from hypothesis import HealthCheck, given, settings
    from hypothesis import strategies as st

    from paper_2305_15163_b200 import binio

    shapes = st.tuples(st.integers(0, 5), st.integers(0, 5))
    names = st.text(min_size=0, max_size=12)

    @settings(max_examples=60, deadline=None,
              suppress_health_check=[HealthCheck.function_scoped_fixture])
    @given(st.lists(st.tuples(names, shapes, st.integers(0, 2 ** 32 - 1)), min_size=0,
                    max_size=6, unique_by=lambda t: t[0]))
    def check(recs):
        mats = []
        for nm, (r, c), seed in recs:
            bits = np.random.default_rng(seed).integers(0, 2 ** 63, size=r * c, dtype=np.int64)
            mats.append((nm, bits.view(np.float64).reshape(r, c)))
        path = tmp_path / "p.bin"
        binio.write_matrices(path, mats)
        got = binio.read_matrices(path)
        assert list(got) == [m[0] for m in mats]
        for nm, a in mats:
            assert got[nm].shape == a.shape
            np.testing.assert_array_equal(got[nm].view(np.uint64), a.view(np.uint64))

    check()
