import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2510_03996_b200 as fh
ctx = fh.SlotContext(fh.ContextConfig.preset("config2"))
steps = [1 << i for i in range(15)] + [-1]
ctx.keygen_rotations(steps)
rng = np.random.default_rng(0)
cts = [fh.SlotVector.encode_top(ctx, rng.uniform(-1, 1, 32768)) for _ in range(8)]
stream = torch.cuda.ExternalStream(ctx.stream())
c = 0
for rep in range(6):
    ctx.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    for s in range(20):
        ts = [steps[(c + b) % 16] for b in range(8)]
        c += 8
        keep = fh.rotate_many(cts, ts)
    h = (time.perf_counter() - h0) * 1e3 / 20
    e1.record(stream); e1.synchronize()
    print(f"rep {rep}: gpu {e0.elapsed_time(e1)/20:.3f} ms/step host {h:.3f} ms/step", flush=True)
import os
print("cpus", os.cpu_count(), open('/proc/loadavg').read().strip())
