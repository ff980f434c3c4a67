import sys, time, tempfile
sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M
from oracle import ref as sref
ring = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 12
spec = M.lenet5(ring=ring, depth_budget=depth)
x = np.random.default_rng(3002).uniform(0, 1, (1, 28, 28))
d = tempfile.mkdtemp()
path = spec.write(d)
rl, rows, rev, rwall = sref.infer(path, x)
t0 = time.time()
em = M.EncryptedModel(spec)
print(f"ring {ring} depth {depth}: bootstraps {em.n_boot} (ref {sum(r[3] for r in rows)}), setup {time.time()-t0:.1f}s, L={em.ctx.L}", flush=True)
r = em.infer(x)  # warm (keygen)
r = em.infer(x, time_layers=True)
r2 = em.infer(x)
print("logits gpu", np.round(r2.logits, 4))
print("logits ref", np.round(rl, 4))
print("max abs err", np.abs(r2.logits - rl).max(), "argmax", int(np.argmax(r2.logits)), int(np.argmax(rl)))
print("wall ms", round(r2.wall_ms, 1), "ref sim ms", round(rwall, 1))
print("ledger equal:", [(a[0], a[2], a[3]) for a in r2.ledger] == [(b[0], b[1], b[2]) for b in rows])
print({k: round(v, 1) for k, v in r.layer_ms.items()})
print(r2.stats)
