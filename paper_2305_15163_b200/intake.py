"""Intake of the reference's own ``RomInstance`` (the drop-in seam).

``RomInstance.from_ddrom(ref)`` turns a ``ddrom.driver.RomInstance`` into the
artifact dictionary the device context uploads -- the same arrays
``tools/make_golden.py`` commits as ``tests/golden/*_artifacts.npz``.
"""

from __future__ import annotations

import json

import numpy as np


def arrays_from_ddrom(inst, full_maps: bool = True) -> dict:
    """Everything the online solve consumes from a reference
    ``ddrom.driver.RomInstance`` (after ``attach_hr`` and
    ``fit_initializer``), extracted the way ``build_problem`` builds it
    (driver.py:356-436): per block the decoder subnet (``extract_subnet``,
    hyper.py:200-222) or the restricted POD basis (pod.py:95-97), the full
    interface decoder (autoencoder.py:104-112), the sampled residual rows and
    local column order of ``RestrictedResidual`` (driver.py:392-396),
    ``CA = C @ A_i`` (driver.py:368-369) or the SRPC ``Ahat_i``
    (driver.py:374-378), gappy weights (hyper.py:153-160), and the fitted RBF
    initializer (driver.py:59-90 with scipy's ``_coeffs/_shift/_scale/
    powers``).  ``full_maps``: also the full interior (and SRPC interface)
    maps for ``RomInstance.decode`` (driver.py:148-152).

    Imports ``ddrom`` lazily: only a caller holding a reference instance
    needs it."""
    from ddrom.autoencoder import Autoencoder
    from ddrom.hyper import extract_subnet, hr_rows_for_subdomain
    from ddrom.pod import LinearMap

    part = inst.partition
    grid = part.grid
    out = {}
    kind = "nm" if isinstance(inst.interior_maps[0], Autoencoder) else "ls"
    srpc = inst.constraint_mode == "srpc"
    n_int = [m.latent_dim for m in inst.interior_maps]
    n_gam = [g.latent_dim for g in inst.interface_maps]
    act = inst.interior_maps[0].activation if kind == "nm" else "linear"
    gam_act = inst.interface_maps[0].activation if kind == "nm" else "linear"
    for i, sub in enumerate(part.subdomains):
        hr = inst.hr[i]
        rows = hr.apply_B_rows()
        io, gio = hr_rows_for_subdomain(part, i, rows)
        cols = np.concatenate([sub.interior_cols[io], sub.interface_cols[gio]])
        p = f"b{i}_"
        out[p + "res_rows"] = sub.res_rows[rows].astype(np.int64)
        out[p + "cols"] = cols.astype(np.int64)
        out[p + "io"] = io.astype(np.int64)
        out[p + "gio"] = gio.astype(np.int64)
        out[p + "n_interior"] = np.int64(sub.n_interior)
        out[p + "n_interface"] = np.int64(sub.n_interface)
        if srpc:   # driver.py:374-378
            out[p + "Ahat"] = inst.rom_constraints.blocks[i].toarray()
        else:      # driver.py:366-373
            out[p + "CA"] = inst.wfpc_C @ inst.fom_constraints.blocks[i].toarray()
        if hr.mode == "gappy":   # hyper.py:107-118,153-160
            out[p + "weights"] = np.ascontiguousarray(hr.weights)
        im, gm = inst.interior_maps[i], inst.interface_maps[i]
        if full_maps:
            # global dof columns of the block (Partition.restrict, partition.py:232-235)
            out[p + "int_cols"] = sub.interior_cols.astype(np.int64)
            out[p + "gam_cols"] = sub.interface_cols.astype(np.int64)
        # the full interior map for RomInstance.decode (driver.py:148-152);
        # left out for the 480^2 / 960^2 instances (the decode is not on the
        # solve path and the maps are ~50 MB per block)
        if kind == "nm" and not full_maps:
            pass
        elif kind == "nm":
            W2f = im.W2g.tocsr()
            out[p + "intf_W1"] = np.ascontiguousarray(im.W1g)
            out[p + "intf_b1"] = im.b1g.copy()
            out[p + "intf_W2_indptr"] = W2f.indptr.astype(np.int64)
            out[p + "intf_W2_indices"] = W2f.indices.astype(np.int64)
            out[p + "intf_W2_data"] = W2f.data.copy()
            out[p + "intf_scale"] = im.norm.scale.copy()
            out[p + "intf_shift"] = im.norm.shift.copy()
        else:
            out[p + "intf_Phi"] = np.ascontiguousarray(im.Phi)
        if srpc:
            # the residual uses the interface map restricted to gio
            # (driver.py:400-402); the full map is kept for the decode
            if kind == "nm":
                W2f = gm.W2g.tocsr()
                out[p + "gamf_W1"] = np.ascontiguousarray(gm.W1g)
                out[p + "gamf_b1"] = gm.b1g.copy()
                out[p + "gamf_W2_indptr"] = W2f.indptr.astype(np.int64)
                out[p + "gamf_W2_indices"] = W2f.indices.astype(np.int64)
                out[p + "gamf_W2_data"] = W2f.data.copy()
                out[p + "gamf_scale"] = gm.norm.scale.copy()
                out[p + "gamf_shift"] = gm.norm.shift.copy()
            else:
                out[p + "gamf_Phi"] = np.ascontiguousarray(gm.Phi)
        if kind == "nm":
            sn = extract_subnet(im, io)
            out[p + "int_W1"] = np.ascontiguousarray(sn.W1)
            out[p + "int_b1"] = sn.b1.copy()
            out[p + "int_W2_indptr"] = sn.W2.indptr.astype(np.int64)
            out[p + "int_W2_indices"] = sn.W2.indices.astype(np.int64)
            out[p + "int_W2_data"] = sn.W2.data.copy()
            out[p + "int_scale"] = sn.scale.copy()
            out[p + "int_shift"] = sn.shift.copy()
            out[p + "int_hidden_idx"] = sn.hidden_idx.astype(np.int64)
            if srpc:
                sg = extract_subnet(gm, gio) if gio.size else None
                H = sg.W1.shape[0] if sg is not None else 0
                out[p + "gam_W1"] = (np.ascontiguousarray(sg.W1) if sg is not None
                                     else np.zeros((0, gm.latent_dim)))
                out[p + "gam_b1"] = sg.b1.copy() if sg is not None else np.zeros(0)
                out[p + "gam_W2_indptr"] = (sg.W2.indptr.astype(np.int64) if sg is not None
                                            else np.zeros(1, np.int64))
                out[p + "gam_W2_indices"] = (sg.W2.indices.astype(np.int64) if sg is not None
                                             else np.zeros(0, np.int64))
                out[p + "gam_W2_data"] = sg.W2.data.copy() if sg is not None else np.zeros(0)
                out[p + "gam_scale"] = sg.scale.copy() if sg is not None else np.zeros(0)
                out[p + "gam_shift"] = sg.shift.copy() if sg is not None else np.zeros(0)
                del H
            else:
                W2g = gm.W2g.tocsr()
                out[p + "gam_W1"] = np.ascontiguousarray(gm.W1g)
                out[p + "gam_b1"] = gm.b1g.copy()
                out[p + "gam_W2_indptr"] = W2g.indptr.astype(np.int64)
                out[p + "gam_W2_indices"] = W2g.indices.astype(np.int64)
                out[p + "gam_W2_data"] = W2g.data.copy()
                out[p + "gam_scale"] = gm.norm.scale.copy()
                out[p + "gam_shift"] = gm.norm.shift.copy()
        else:
            assert isinstance(im, LinearMap) and isinstance(gm, LinearMap)
            out[p + "int_Phi"] = np.ascontiguousarray(im.restrict_outputs(io).Phi)
            out[p + "gam_Phi"] = np.ascontiguousarray(
                gm.restrict_outputs(gio).Phi if srpc else gm.Phi)
    ini = inst.initializer
    rbf = ini._rbf
    meta = {
        "kind": kind, "activation": act, "gam_activation": gam_act,
        "constraint": inst.constraint_mode, "hr": inst.hr[0].mode,
        "nx": grid.nx, "ny": grid.ny,
        "nu": grid.nu, "nsub_x": part.nsub_x, "nsub_y": part.nsub_y,
        "nblocks": len(part.subdomains), "n_int": n_int, "n_gam": n_gam,
        "n_c": int(inst.n_mult), "ndof": int(grid.ndof), "rbf_kernel": rbf.kernel,
        "rbf_epsilon": float(rbf.epsilon),
        "provenance": {k: (v if isinstance(v, (int, float, str)) else str(v))
                       for k, v in inst.provenance.items()},
    }
    out["rbf_lo"] = ini.lo.copy()
    out["rbf_hi"] = ini.hi.copy()
    out["rbf_y"] = np.ascontiguousarray(rbf.y)
    out["rbf_coeffs"] = np.ascontiguousarray(rbf._coeffs)
    out["rbf_shift"] = np.asarray(rbf._shift, dtype=float)
    out["rbf_scale"] = np.asarray(rbf._scale, dtype=float)
    out["rbf_powers"] = np.asarray(rbf.powers, dtype=np.int64)
    out["meta_json"] = np.array(json.dumps(meta))
    return out
