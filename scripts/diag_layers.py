import sys, numpy as np
sys.path.insert(0, '.')
import paper_2510_03996_b200 as fh
from oracle import ref as sref
from tests.test_gpu_layers import run_both, LOGN, DEPTH
cfg = fh.ContextConfig(1 << LOGN, 1 << (LOGN - 1), DEPTH, fh.CryptoMetadata(52, 40, 3), limbs=DEPTH + 1,
                       special_limbs=4, special_bits=60, seed=9001)
ctx = fh.SlotContext(cfg)
ref = sref.Ref(1 << LOGN, 1 << (LOGN - 1), DEPTH)
rng = np.random.default_rng(0)
def rep(tag, out, ev, r):
    got = out.slots()
    err = np.abs(got - r.slots).max()
    bad = np.where(np.abs(got - r.slots) > 1e-3)[0]
    print(f"{tag:40s} err={err:.3g} lvl {out.level()} vs {r.level} trace_eq={ev == r.events} nbad={bad.size} first={bad[:5]}", flush=True)
W, C = 4, 3
x = rng.uniform(-1, 1, (C, W, W))
# primitives
v = x.reshape(-1)
for t in [1, -1, 4, 16]:
    out, ev, r = run_both(ctx, lambda s: fh.rotate(s, t), lambda s: ref.backend_op(0, s, DEPTH, t=t), v); rep(f"rotate {t}", out, ev, r)
m = rng.uniform(-1,1,ctx.slots())
out, ev, r = run_both(ctx, lambda s: fh.mult_plain(s, m), lambda s: ref.backend_op(3, s, DEPTH, b=m), v); rep("mult_plain", out, ev, r)
mask = np.zeros(ctx.slots()); mask[:4] = 1
out, ev, r = run_both(ctx, lambda s: fh.mult_plain(s, mask), lambda s: ref.backend_op(3, s, DEPTH, b=mask), v); rep("mult_plain mask", out, ev, r)
for P in [1, 2]:
    out, ev, r = run_both(ctx, lambda s: fh.pad_input(fh.PackedTensor(s, C, W), P).data, lambda s: ref.pad_input(s, DEPTH, C, W, P), x); rep(f"pad {P}", out, ev, r)
for (WW, S, var) in [(4,2,0),(8,2,1),(8,2,0),(6,2,1)]:
    xx = rng.uniform(-1,1,(1,WW,WW))
    fn = fh.stride_extract_v2 if var else fh.stride_extract_v1
    out, ev, r = run_both(ctx, lambda s: fn(s, WW, S), lambda s: ref.stride(s, DEPTH, WW, S, 0, var), xx); rep(f"stride {WW} {S} {var}", out, ev, r)
for (k,S,P,var) in [(2,1,0,0),(3,1,0,0),(2,2,0,0),(2,2,0,1),(3,1,1,0)]:
    F=2; w = rng.uniform(-1,1,(F,C,k,k)); b = rng.uniform(-1,1,F)
    cc = fh.ConvConfig(C,F,k,S,P,fh.ConvMode.generic,fh.StrideVariant(var))
    out, ev, r = run_both(ctx, lambda s: fh.convolution(fh.PackedTensor(s, C, W), cc, fh.KernelTensor(w,b)).data,
                          lambda s: ref.convolution(s, DEPTH, C, W, F, k, S, P, 0, var, w, b), x); rep(f"conv k{k} S{S} P{P} v{var}", out, ev, r)
