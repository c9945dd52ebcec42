"""binio: the reference's bit-exact matrix format (binio.py:1-87), read and
written by the C++ side of libddnm.so, plus instance files that feed a GPU
context without Python (``ddnm_ctx_create_binio``) and the reference's
serialized nets (``save_net`` / ``load_net``, autoencoder.py:424-479).

Layout: magic ``DDNMROM1``; per record a u32 name length, the UTF-8 name, u64
rows, u64 cols and rows*cols float64 in column-major order, little-endian.
Same errors as the reference: :class:`FormatError` for a bad magic, a
truncated record or a record overrunning the file.
"""

from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import FormatError

INSTANCE_FORMAT = "ddnm-instance-1"

# artifact arrays holding indices (stored as float64, as the reference stores
# CSR indices in save_net, autoencoder.py:435-441)
_INT_SUFFIXES = ("_indptr", "_indices", "res_rows", "_cols", "_io", "_gio", "hidden_idx",
                 "rbf_powers", "n_interior", "n_interface")


def _check(rc: int):
    if rc == -5:
        raise FormatError(N.lib().ddnm_last_error().decode(errors="replace"))
    N.check(rc)


def read_matrices(path) -> dict:
    """binio.read_matrices (binio.py:43-70): ``{name: 2-D float64 array}``."""
    L = N.lib()
    h = C.c_void_p()
    _check(L.ddnm_binio_read(str(path).encode(), C.byref(h)))
    try:
        n = C.c_int64()
        _check(L.ddnm_binio_count(h, C.byref(n)))
        out = {}
        for i in range(n.value):
            name, nlen = C.c_void_p(), C.c_int64()
            r, c = C.c_int64(), C.c_int64()
            d = C.POINTER(C.c_double)()
            _check(L.ddnm_binio_entry(h, i, C.byref(name), C.byref(nlen), C.byref(r), C.byref(c),
                                      C.byref(d)))
            cnt = r.value * c.value
            flat = (np.ctypeslib.as_array(d, shape=(cnt,)).copy() if cnt
                    else np.zeros(0))
            key = C.string_at(name, nlen.value).decode("utf-8") if nlen.value else ""
            out[key] = flat.reshape((r.value, c.value), order="F")
        return out
    finally:
        L.ddnm_binio_free(h)


def write_matrices(path, matrices) -> None:
    """binio.write_matrices (binio.py:22-40): 1-D arrays become one column."""
    items = list(matrices.items() if hasattr(matrices, "items") else matrices)
    names, rows, cols, bufs = [], [], [], []
    for name, arr in items:
        a = np.asarray(arr, dtype=float)
        if a.ndim == 1:
            a = a[:, None]
        if a.ndim != 2:
            raise ValueError(f"matrix {name!r} must be 1-D or 2-D")
        f = np.asfortranarray(a, dtype="<f8")
        names.append(name.encode("utf-8"))
        rows.append(a.shape[0])
        cols.append(a.shape[1])
        bufs.append(f)
    n = len(items)
    cn = (C.c_char_p * n)(*names)
    cl = (C.c_int64 * n)(*[len(b) for b in names])
    cr = (C.c_int64 * n)(*rows)
    cc = (C.c_int64 * n)(*cols)
    cd = (C.POINTER(C.c_double) * n)(*[b.ctypes.data_as(C.POINTER(C.c_double)) for b in bufs])
    _check(N.lib().ddnm_binio_write(str(path).encode(), n, cn, cl, cr, cc, cd))


def write_meta(path, entries: dict) -> None:
    """binio.write_meta (binio.py:73-76)."""
    Path(path).write_text("".join(f"{k} = {v}\n" for k, v in entries.items()),
                          encoding="utf-8")


def read_meta(path) -> dict:
    """binio.read_meta (binio.py:79-87)."""
    out = {}
    for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), 1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if "=" not in line:
            raise FormatError(f"{path}:{lineno}: expected 'key = value'")
        k, v = line.split("=", 1)
        out[k.strip()] = v.strip()
    return out


def load_net(path) -> dict:
    """The reference's serialized autoencoder (save_net, autoencoder.py:424-450:
    ``<path>`` binio + ``<stem>.txt`` header), as the arrays of its decoder:
    ``W1`` (= W1g, hidden x latent), ``b1``, the CSR ``W2_indptr`` /
    ``W2_indices`` / ``W2_data`` (outputs x hidden), ``scale`` / ``shift``
    (normalization), ``activation``, ``band``, ``shift_mask``, dims."""
    path = Path(path)
    m = read_matrices(path)
    hdr = read_meta(path.with_suffix(".txt"))
    need = ("W1g", "b1g", "W2g_data", "W2g_indices", "W2g_indptr", "norm_shift", "norm_scale")
    for k in need:
        if k not in m:
            raise FormatError(f"{path}: missing record {k!r}")
    N_out, width = int(hdr["ambient_dim"]), int(hdr["width"])
    indptr = m["W2g_indptr"].ravel().astype(np.int64)
    if indptr.size != N_out + 1:
        raise FormatError(f"{path}: W2g_indptr does not match ambient_dim")
    return {
        "W1": np.ascontiguousarray(m["W1g"]), "b1": m["b1g"].ravel(),
        "W2_indptr": indptr, "W2_indices": m["W2g_indices"].ravel().astype(np.int64),
        "W2_data": m["W2g_data"].ravel(), "scale": m["norm_scale"].ravel(),
        "shift": m["norm_shift"].ravel(), "activation": hdr["activation"],
        "band": int(hdr["mask_band"]), "shift_mask": int(hdr["mask_shift"]),
        "ambient_dim": N_out, "latent_dim": int(hdr["latent_dim"]), "width": width,
    }


def save_instance(instance, path) -> None:
    """Write a RomInstance's artifacts as an instance file pair: ``path``
    (binio, one record per artifact array) and ``<stem>.txt`` (meta), which
    ``ddnm_ctx_create_binio`` reads without Python."""
    path = Path(path)
    a, m = instance.arrays, instance.meta
    mats = [(k, np.asarray(v)) for k, v in a.items() if k != "meta_json"]
    write_matrices(path, [(k, v.astype(float).reshape(-1) if v.ndim < 2 else v) for k, v in mats])
    meta = {
        "format": INSTANCE_FORMAT, "kind": m["kind"],
        "activation": m.get("activation", "swish"),
        "gam_activation": m.get("gam_activation", m.get("activation", "swish")),
        "constraint": m.get("constraint", "wfpc"), "hr": m.get("hr", "collocation"),
        "nx": m["nx"], "ny": m["ny"], "nu": repr(float(m["nu"])), "nblocks": m["nblocks"],
        "n_int": ",".join(str(int(v)) for v in m["n_int"]),
        "n_gam": ",".join(str(int(v)) for v in m["n_gam"]),
        "n_c": m["n_c"], "rbf_kernel": m.get("rbf_kernel", "thin_plate_spline"),
        "rbf_epsilon": repr(float(m.get("rbf_epsilon", 1.0))),
        "meta_json": json.dumps(m),
        # array ranks (binio stores matrices; 1-D arrays are single columns)
        "vectors": ",".join(k for k, v in mats if v.ndim == 1),
        "scalars": ",".join(k for k, v in mats if v.ndim == 0),
    }
    write_meta(path.with_suffix(".txt"), meta)


def load_instance_arrays(path) -> dict:
    """Inverse of :func:`save_instance`: the artifact dictionary RomInstance
    takes (indices back to int64, vectors back to 1-D, scalars to 0-d)."""
    path = Path(path)
    meta = read_meta(path.with_suffix(".txt"))
    if meta.get("format") != INSTANCE_FORMAT:
        raise FormatError(f"{path.with_suffix('.txt')}: not a {INSTANCE_FORMAT} meta file")
    vec = set(filter(None, meta.get("vectors", "").split(",")))
    sca = set(filter(None, meta.get("scalars", "").split(",")))
    out = {}
    for k, v in read_matrices(path).items():
        if k in vec:
            v = v[:, 0]
        elif k in sca:
            v = v.reshape(())
        if k.endswith(_INT_SUFFIXES):
            v = v.astype(np.int64)
        out[k] = v
    out["meta_json"] = np.array(meta["meta_json"])
    return out
