DDNM_PROF=1 python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import paper_2305_15163_b200 as P
inst = P.RomInstance.load('tests/golden/c0_nm_artifacts.npz')
mu = P.seeded_parameters(4096, seed=1000)
for _ in range(2): r = P.solve_rom_batch(inst, mu)
prof = inst.context().profile(); tot = sum(prof.values()) or 1
print({k: f"{100*v/tot:.1f}%" for k, v in prof.items()})
print(r.seconds*1e3, r.rounds)
PY
