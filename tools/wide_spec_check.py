"""Speculative step lengths do not change results: DDNM_WIDE=1 with and
without DDNM_WIDE_NOSPEC, and a sub-batch vs the whole batch (bitwise)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2305_15163_b200 as P
    name, B = sys.argv[2], int(sys.argv[3])
    inst = P.RomInstance.load(os.path.join(ROOT, "tests", "golden", f"{name}_artifacts.npz"))
    mu = P.seeded_parameters(B, seed=1000)
    r = P.solve_rom_batch(inst, mu)
    r2 = P.solve_rom_batch(inst, mu[: B // 3])
    np.savez(sys.argv[4], x=r.x, lam=r.lam, n_iter=r.n_iter, n_evals=r.n_evals, status=r.status,
             x2=r2.x, lam2=r2.lam, n_evals2=r2.n_evals, sec=r.seconds)
    sys.exit(0)

name = sys.argv[1] if len(sys.argv) > 1 else "c0_nm"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
out = {}
for tag, env in (("spec", {}), ("nospec", {"DDNM_WIDE_NOSPEC": "1"})):
    e = dict(os.environ, DDNM_WIDE="1", **env)
    f = f"/tmp/wsc_{tag}.npz"
    subprocess.run([sys.executable, __file__, "child", name, str(B), f], check=True, env=e)
    out[tag] = np.load(f)
a, b = out["spec"], out["nospec"]
for k in ("x", "lam", "n_iter", "n_evals", "status"):
    print(k, "spec == nospec:", bool(np.array_equal(a[k], b[k])))
n = B // 3
print("sub-batch == batch (spec):", bool(np.array_equal(a["x2"], a["x"][:n])), bool(np.array_equal(a["lam2"], a["lam"][:n])),
      bool(np.array_equal(a["n_evals2"], a["n_evals"][:n])))
print(f"seconds spec {float(a['sec'])*1e3:.2f} ms, nospec {float(b['sec'])*1e3:.2f} ms")
