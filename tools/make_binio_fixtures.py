"""Reference-written binio fixtures (run in the build container only; imports
the reference from /root/reference/pkg/src -- nothing on the GPU box reads it).

* tests/golden/ref_binio_matrices.bin (+ .npz with the same arrays): written
  by ddrom.binio.write_matrices (binio.py:22-40): 1-D, 2-D, empty, special
  values (signed zero, inf, nan, subnormal), a UTF-8 name;
* tests/golden/ref_net_int0.bin / .txt: ddrom.autoencoder.save_net
  (autoencoder.py:424-450) of the tiny instance's interior net 0, whose full
  decoder is b0_intf_* of tests/golden/tiny_nm_artifacts.npz.
"""
import os
import pickle
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def main():
    from ddrom import binio
    from ddrom.autoencoder import save_net
    mats = {
        "vec": np.array([1.5, -2.0, 0.0, -0.0, np.inf, -np.inf, 5e-324, 1e308]),
        "mat": np.arange(12, dtype=float).reshape(3, 4) * np.pi,
        "empty": np.zeros((0, 3)),
        "nan": np.array([[np.nan]]),
        "ünicode_name": np.array([[7.0, 8.0]]),
    }
    binio.write_matrices(os.path.join(GOLD, "ref_binio_matrices.bin"), mats)
    np.savez(os.path.join(GOLD, "ref_binio_matrices.npz"),
             **{f"m{i}": v for i, v in enumerate(mats.values())},
             names=np.array(list(mats.keys())))
    with open(os.path.join(ROOT, "artifacts_cache", "tiny_nm.pkl"), "rb") as f:
        inst = pickle.load(f)
    save_net(os.path.join(GOLD, "ref_net_int0.bin"), inst.interior_maps[0])
    print("written")


if __name__ == "__main__":
    main()
