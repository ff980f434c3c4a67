import sys, time, tempfile
sys.path.insert(0, '.')
import numpy as np
from paper_2510_03996_b200 import model as M
from oracle import ref as sref
depth = int(sys.argv[1]) if len(sys.argv) > 1 else 12
ring = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
def norm(x):
    return (x - 0.5) / 0.2887
spec = M.resnet20(ring=ring, depth_budget=depth)
cal = [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]
spec = M.calibrate_relu_scales(spec, cal)
x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
path = spec.write(tempfile.mkdtemp())
t0 = time.time(); rl, rows, rev, rwall = sref.infer(path, x); print("ref infer s", round(time.time() - t0, 2), flush=True)
t0 = time.time()
em = M.EncryptedModel(spec)
print(f"bootstraps {em.n_boot} (ref {sum(r[3] for r in rows)}), setup {time.time()-t0:.1f}s L={em.ctx.L}", flush=True)
t0 = time.time(); r = em.infer(x, time_layers=True); print("first infer s", round(time.time() - t0, 2), flush=True)
t0 = time.time(); r2 = em.infer(x); print("second infer s", round(time.time() - t0, 2), flush=True)
print("logits gpu", np.round(r2.logits, 4))
print("logits ref", np.round(rl, 4))
print("max abs err", np.abs(r2.logits - rl).max(), "argmax", int(np.argmax(r2.logits)), int(np.argmax(rl)))
print("ledger equal:", [(a[0], a[2], a[3]) for a in r2.ledger] == [(b[0], b[1], b[2]) for b in rows])
top = sorted(r.layer_ms.items(), key=lambda kv: -kv[1])[:12]
print("top layers ms", [(k, round(v)) for k, v in top])
print(r2.stats, "keys", em.ctx.key_count())
