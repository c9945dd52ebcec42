"""Build the SRPC and gappy-HR variants of the cached reference instances
 with the *reference* package (offline, build container).

From ``artifacts_cache/<tag>_snap.pkl`` and ``<tag>_nm.pkl`` (written by
``tools/make_artifacts.py``) this writes

* ``<tag>_nmg.pkl``  -- the same NM-ROM with gappy HR instead of collocation:
  ``fit_initializer(attach_hr(nm, snap, "gappy", n_samples, 1e-10), snap)``
  (driver.py:283-300, hyper.py:153-160);
* ``<tag>_srpc.pkl`` -- the NM-ROM with strong ROM-port constraints: the
  interior nets of ``<tag>_nm`` (``train_nets`` trains them with the same
  seeds in both modes, driver.py:238-240) plus Sigmoid port nets trained
  exactly as ``train_nets`` does for srpc (seed offset 300 + port,
  port_band=3, port_shift=3; driver.py:247-250), assembled as
  ``build_nmrom`` does (driver.py:273-279), collocation HR and the RBF
  initializer;
* ``<tag>_lsg.pkl`` / ``<tag>_lss.pkl`` -- the LS-ROM with gappy HR and the
  SRPC LS-ROM (``build_lsrom(..., "srpc")``, driver.py:208-217).
"""

from __future__ import annotations

import argparse
import os
import pickle
import sys
import time
from dataclasses import replace
from multiprocessing import get_context

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SETTINGS = {   # tag: (n_samples, epochs, ls_dims)
    "tiny": (40, 2000, (8, 4)),
    "c0": (180, 2000, (20, 8)),
}


def _train_port(args):
    from ddrom.autoencoder import TrainConfig, build_mask, train
    X, n, offset, band, shift, epochs, seed = args
    cfg = replace(TrainConfig(epochs=epochs, seed=seed), seed=seed + offset)
    n_eff = max(1, min(n, X.shape[0] - 1))
    t0 = time.time()
    ae, _ = train(X, build_mask(X.shape[0], band, shift), n_eff, cfg, activation="sigmoid")
    return ae, time.time() - t0


def main():
    from ddrom.autoencoder import assemble_srpc_interface
    from ddrom.driver import (RomInstance, attach_hr, build_lsrom, fit_initializer,
                              port_latent_dims)
    from ddrom.partition import assemble_rom_constraints

    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="tiny", choices=sorted(SETTINGS))
    ap.add_argument("--cache", default=os.path.join(ROOT, "artifacts_cache"))
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--only", nargs="*", default=["nmg", "srpc", "lsg", "lss"])
    a = ap.parse_args()
    n_samples, epochs, ls_dims = SETTINGS[a.tag]
    with open(os.path.join(a.cache, f"{a.tag}_snap.pkl"), "rb") as f:
        snap = pickle.load(f)
    with open(os.path.join(a.cache, f"{a.tag}_nm.pkl"), "rb") as f:
        nm = pickle.load(f)
    part = nm.partition
    n_gam = nm.provenance["n_gam"]
    t0 = time.time()

    def dump(inst, name):
        with open(os.path.join(a.cache, f"{a.tag}_{name}.pkl"), "wb") as f:
            pickle.dump(inst, f)
        print(f"[{a.tag}_{name}] written ({time.time() - t0:.1f}s)", flush=True)

    if "nmg" in a.only:
        dump(fit_initializer(attach_hr(nm, snap, "gappy", n_samples=n_samples,
                                       energy=1e-10), snap), "nmg")
    if "srpc" in a.only:
        dims = port_latent_dims(part.ports, n_gam)
        jobs = [(snap.port[j], dims[j], 300 + j, 3, 3, epochs, 0) for j in dims]
        with get_context("fork").Pool(min(a.procs, len(jobs))) as pool:
            res = pool.map(_train_port, jobs)
        nets = {j: r[0] for j, r in zip(dims, res)}
        print(f"[{a.tag}_srpc] port nets trained: "
              f"{[round(r[1], 1) for r in res]} s", flush=True)
        gams = [assemble_srpc_interface(part.ports, nets, i)
                for i in range(len(part.subdomains))]
        pdims = {j: net.latent_dim for j, net in nets.items()}
        prov = {"rom": "nmrom", "constraint": "srpc", "hr": "none",
                "n_int": nm.provenance["n_int"], "n_gam": n_gam, "seed": 0}
        srpc = RomInstance(partition=part, interior_maps=list(nm.interior_maps),
                           interface_maps=gams, constraint_mode="srpc",
                           rom_constraints=assemble_rom_constraints(part.ports, pdims),
                           provenance=prov)
        dump(fit_initializer(attach_hr(srpc, snap, "collocation", n_samples=n_samples,
                                       energy=1e-10), snap), "srpc")
    if "lsg" in a.only:
        with open(os.path.join(a.cache, f"{a.tag}_ls.pkl"), "rb") as f:
            ls = pickle.load(f)
        dump(fit_initializer(attach_hr(ls, snap, "gappy", n_samples=n_samples,
                                       energy=1e-10), snap), "lsg")
    if "lss" in a.only:
        lss = build_lsrom(part, snap, ls_dims[0], ls_dims[1], "srpc")
        dump(fit_initializer(attach_hr(lss, snap, "collocation", n_samples=n_samples,
                                       energy=1e-10), snap), "lss")


if __name__ == "__main__":
    main()
