#!/usr/bin/env python
"""bench.py -- FHEON hot path on B200: encrypted ResNet-20 inference, s/image.

Headline (BASELINE.json metric "encrypted inference s/image (1 B200)", configs[3]):
ResNet-20 on a 3x32x32 input (seeded U[0,1], per-channel normalised), 3x3 convs
at 16/32/64 channels, three stages of three basic blocks with 2x2/s2
downsampling, global avgpool, FC 64->10, He-normal weights (seed 4001),
degree-59 Chebyshev ReLU with calibrated frozen scales, CKKS N = 2^16 with full
bootstrapping -- at 128-bit security (HE standard, uniform ternary secret,
log2 QP <= 1747; bootstrapping through the sparse-secret encapsulation).  One
step = one encrypted inference through every layer and bootstrap.

  value  s/image with the encrypted input resident in HBM: the forward pass
         (every layer + bootstrap on the GPU) timed with CUDA events on the
         engine stream, max over ranks; value = time / images of all ranks
  e2e    the repo's public API EncryptedModel.infer(): host image -> encode +
         encrypt -> forward -> decrypt -> host logits, wall clock per image,
         image coefficients up and two decrypted limbs down declared
  roofline  the NTT (the largest kernel class of the step, integer-pipe bound)
         timed live with CUDA events in a second pass of the same steps:
         butterflies/s against the measured lazy-Shoup butterfly peak
  cpu_baseline  the reference's own infer() (oracle/_ref: the unmodified slotcnn
         core) on the same spec, weights and input, one host core
  rotations  BASELINE configs[1] key-switch rotation microbench (N=2^16, L=24,
         dnum 3): rotations/s device and end to end, k_ks_inner HBM roofline,
         tensor-core basis conversion, the C2 primitive sweep
  models  LeNet-5 / ResNet-20 / VGG-16 variants (reference specs, insecure
         reference-preset chains, reference rotation schedule) with their logit
         error against the reference's infer() and a security disclosure each

`--impl reference` times the reference's own infer() (oracle/_ref) on the same
spec, weights and input: 1-thread latency (value) and all-core throughput.
Multi-GPU: independent replicas, weak scaling.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LOGN, L, K, DNUM = 16, 24, 8, 3
N = 1 << LOGN
S = N // 2
NKEYS = 16
CONFIG = {"workload": "configs[1] CKKS key-switch rotation", "ring_dimension": N, "slots": S, "limbs": L,
          "special_limbs": K, "dnum": DNUM, "prime_bits": "60 + 23x50, special 8x60",
          "rotation_steps": "2^0..2^14 and -1 (16 keys, one per rotation, cycled)", "level": L - 1,
          "l2": "inputs larger than L2 (8 x 25 MiB ciphertexts + 1.5 GiB keys), no flush"}
HEAD_DEPTH = 11  # ResNet-20 depth budget of the 128-bit headline chain (fastest of 8..14 measured)


def head_config(depth):
    """The `config` both arms print for the headline (identical dicts: same_config)."""
    return {"workload": "configs[3] ResNet-20 encrypted inference", "model": "resnet20 (BASELINE configs[3])",
            "ring_dimension": N, "slots": S, "depth_budget": depth, "global_batch": 1,
            "input": "3x32x32 U[0,1] seed 4001, per-channel normalised (x - 0.5) / 0.2887",
            "weights": "He-normal seed 4001 (paper_2510_03996_b200.model.resnet20), bias 0",
            "relu": "degree-59 Chebyshev, scales calibrated on seeds 4002..4007 and frozen",
            "downsampling": "2x2/s2 conv + projection (models/resnet20.json)",
            "l2": "working set (keys ~37 GB) far above the 126 MB L2, no flush", "parallelism": "replicas"}


def head_spec(depth):
    from paper_2510_03996_b200 import model as M

    def norm(x):
        return (x - 0.5) / 0.2887

    cal = [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]
    spec = M.calibrate_relu_scales(M.resnet20(ring=N, depth_budget=depth), cal)
    x = norm(np.random.default_rng(4001).uniform(0, 1, (3, 32, 32)))
    return spec, x


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        if os.environ.get("FHEON_NO_CLOCKS"):
            return self
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("FHEON_CLOCKS_MS", "500")], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


def measured_peak_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def committed_traffic():
    """dram bytes per launch of the roofline kernel from the committed ncu --set full capture."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        return d.get("ks_inner_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------- configs[1] rotation microbench
def rotation_bench(args):
    """BASELINE configs[1] key-switch rotations (the round-1 headline, kept as an
    extra block): device rotations/s, end to end through the packed wire format,
    k_ks_inner HBM roofline, NTT / tensor-core basis-conversion shares, C2 sweep."""
    import torch
    import paper_2510_03996_b200 as fh
    from paper_2510_03996_b200 import replicas

    ws, rank, local = dist_env()
    B = args.batch
    ctx = fh.SlotContext(fh.ContextConfig.preset("config2"))
    steps_pow = [1 << i for i in range(NKEYS - 1)] + [-1]
    ctx.keygen_rotations(steps_pow)
    ctx.set_strict_keys(True)
    rng = np.random.default_rng(2001 + rank)
    cts = [fh.SlotVector.encode_top(ctx, rng.uniform(-1, 1, S)) for _ in range(B)]
    stream = torch.cuda.ExternalStream(ctx.stream())
    counter = [0]

    def step():
        # B independent rotations (distinct ciphertexts, distinct keys) in one
        # batched key-switch pipeline through the public API
        ts = []
        for b in range(B):
            ts.append(steps_pow[counter[0] % NKEYS])
            counter[0] += 1
        return fh.rotate_many(cts, ts)

    def barrier():
        torch.cuda.synchronize()
        ctx.sync()
        if ws > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    barrier()
    st0 = ctx.stats()
    # FHEON_PROFILE_RANGE=1: limit an `ncu --profile-from-start off` capture to the timed steps
    prof = None
    if os.environ.get("FHEON_PROFILE_RANGE"):
        import ctypes
        prof = ctypes.CDLL("libcudart.so.12")
        prof.cudaProfilerStart()
    ctx.timer_arm(1)  # key-switch inner product, timed live in the region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        keep = None
        h0 = time.perf_counter()
        for _ in range(args.steps):
            keep = step()
        host_ms = (time.perf_counter() - h0) * 1e3
        e1.record(stream)
        e1.synchronize()
    ms = e0.elapsed_time(e1)
    if prof is not None:
        prof.cudaProfilerStop()
    ks_ms, ks_n = ctx.timer_read()
    ctx.timer_arm(0)
    st1 = ctx.stats()
    del keep
    barrier()
    value, ms_max = replicas.replica_throughput(ms, args.steps * B, torch.device("cuda", local))

    # ---- the NTT's share and integer roofline inside the same step (second
    # pass of K steps with the NTT class timed live; every limb-NTT is
    # (N/2) log2 N lazy Shoup butterflies)
    n0 = ctx.stats()["ntt_limbs"]
    ctx.timer_arm(2)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        keep = step()
    f1.record(stream)
    f1.synchronize()
    ms_ntt_pass = f0.elapsed_time(f1)
    ntt_ms, ntt_n = ctx.timer_read()
    ctx.timer_arm(0)
    del keep
    ntt_limbs = ctx.stats()["ntt_limbs"] - n0
    bfly = ntt_limbs * (N // 2) * LOGN
    try:
        bpeak = json.load(open(os.path.join(ROOT, "profiles", "int_peak.json")))["shoup_ct_butterflies_per_s"]
        bsrc = "measured (profiles/int_peak.json: lazy Shoup butterfly, IMAD.WIDE-bound)"
    except Exception:
        bpeak, bsrc = 8.7e11, "fallback"
    ntt_rate = bfly / (ntt_ms / 1e3)
    roofline_ntt = {"kernel": "ntt_phase_kernel (COL + ROW phases, forward and inverse)", "bound": "int",
                    "achieved": round(ntt_rate / 1e9, 1), "peak": round(bpeak / 1e9, 1), "unit": "Gbutterfly/s",
                    "frac": round(ntt_rate / bpeak, 4), "peak_source": bsrc, "limb_ntts_per_step":
                    ntt_limbs // max(1, args.steps), "share_of_step": round(ntt_ms / ms_ntt_pass, 4),
                    "hbm_gbs": round(ntt_limbs * N * 8 * 4 / (ntt_ms / 1e3) / 1e9, 1)}

    # ---- the tensor-core basis conversions (ModUp class 3, ModDown class 4),
    # timed live in two more passes.  Algorithmic work: exact 64x64-bit
    # products, per rotation sum_j (L + K - alpha_j) alpha_j (ModUp) + 2 L K
    # (ModDown) per coefficient; each is 8 x 16 int8 MACs on the tensor cores.
    bc_ms = {}
    for cls in (3, 4):
        ctx.timer_arm(cls)
        for _ in range(args.steps):
            keep = step()
        torch.cuda.synchronize()
        bc_ms[cls], _ = ctx.timer_read()
        ctx.timer_arm(0)
        del keep
    alpha = (L + DNUM - 1) // DNUM
    digs = [min(alpha, L - j * alpha) for j in range((L + alpha - 1) // alpha)]
    macs_rot = (sum((L + K - a) * a for a in digs) + 2 * L * K) * N
    bc_rate = macs_rot * args.steps * B / ((bc_ms[3] + bc_ms[4]) / 1e3)
    int8_peak = 2 * json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] * 1e12 / 2 \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 2.25e15
    roofline_bconv = {"kernel": "k_bconv_tc (ModUp + ModDown basis conversion, tcgen05.mma kind::i8)",
                      "bound": "tensor", "achieved": round(bc_rate / 1e12, 3),
                      "peak": round(int8_peak / 128 / 1e12, 3), "unit": "T exact 64-bit MAC/s",
                      "frac": round(bc_rate / (int8_peak / 128), 4),
                      "peak_source": "2 x measured bf16 dense (MEASURED_PEAKS.json) int8 MAC/s / 128 int8 MACs "
                                     "per 64-bit product (8 bytes x 16 shift columns)",
                      "cuda_core_roofline": 1.29,
                      "cuda_core_roofline_note": "17.75 IMAD.WIDE.U32/clk/SM (profiles/int_peak.json) / 4 per "
                                                 "64x64->128 product, 148 SMs at 1965 MHz",
                      "share_of_step": round((bc_ms[3] + bc_ms[4]) / ms, 4),
                      "macs_per_rotation": macs_rot}

    # ---- roofline of the key-switch inner product (per launch: one rotation)
    E = L + K
    beta = (L + (L + DNUM - 1) // DNUM - 1) // ((L + DNUM - 1) // DNUM)
    per_rot = (beta * E * N + 2 * beta * E * N + 2 * E * N) * 8  # digits + key (read), acc (write)
    rot_per_launch = args.steps * B / max(1, ks_n)  # one launch covers the step's batch of rotations
    alg_bytes = int(per_rot * rot_per_launch)
    ks_avg_ms = ks_ms / max(1, ks_n)
    achieved = alg_bytes / (ks_avg_ms / 1e3) / 1e9
    peak, peak_kind = measured_peak_hbm()

    # ---- e2e through the C ABI with host buffers (pinned)
    # ciphertexts cross PCIe in the packed wire format (fheon_ct_*_packed: b_i =
    # bit_length(q_i) bits per word, 0.79 of the raw u64 words at this chain);
    # the host copies are made once, untimed, by the engine's own packed download
    PW = ctx.packed_words(L)
    host_in = [torch.empty(PW, dtype=torch.uint64, pin_memory=True).numpy() for _ in range(B)]
    host_out = [torch.empty(PW, dtype=torch.uint64, pin_memory=True).numpy() for _ in range(B)]
    for b in range(B):
        cts[b].packed(out=host_in[b])
    scale = cts[0].scale()

    host_out2 = [torch.empty(PW, dtype=torch.uint64, pin_memory=True).numpy() for _ in range(B)]
    parity = [0]

    def e2e_step():
        # pinned packed host words -> device (upload stream: copy + unpack kernel),
        # rotations (compute stream), pack kernel + device -> pinned host (download
        # stream): consecutive steps overlap
        outs = host_out if parity[0] == 0 else host_out2
        parity[0] ^= 1
        xs = [fh.SlotVector.from_packed(ctx, host_in[b], L, scale, async_copy=True) for b in range(B)]
        ts = []
        for b in range(B):
            ts.append(steps_pow[counter[0] % NKEYS])
            counter[0] += 1
        for b, y in enumerate(fh.rotate_many(xs, ts)):
            y.packed(out=outs[b], async_copy=True)

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    # three timed windows, the median reported: one window is a few hundred ms of PCIe
    # traffic, and a transient host stall (page-in, another process) would otherwise
    # decide the number
    e2e_steps = max(3, args.steps // 2)
    windows = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_step()
        barrier()
        v, _ = replicas.replica_throughput((time.perf_counter() - t0) * 1e3, e2e_steps * B,
                                           torch.device("cuda", local))
        windows.append(v)
    e2e_val = float(np.median(windows))
    ct_bytes = PW * 8

    extras = {}
    if rank == 0 and not args.quick:
        extras = primitives(ctx, fh)
    line = {
        "metric": "rotations/s (CKKS key-switch rotation, N=2^16, L=24, dnum=3)",
        "value": round(value, 1),
        "unit": "rotations/s",
        "steps": args.steps,
        "ms_per_step": round(ms_max / args.steps, 4),
        "host_enqueue_ms_per_step": round(host_ms / args.steps, 4),
        "security": fh.host_security(fh.ContextConfig.preset("config2")),
        "config": dict(CONFIG, batch_per_step=B, parallelism=f"replicas x{ws}"),
        "e2e": {"value": round(e2e_val, 1), "unit": "rotations/s", "h2d_bytes_per_step": B * ct_bytes,
                "d2h_bytes_per_step": B * ct_bytes,
                "path": "C ABI: fheon_ct_upload_packed_async (pinned packed wire format, upload stream, "
                        "unpacked on the device) -> fheon_rotate_many -> fheon_ct_download_packed_async "
                        "(packed on the device, download stream); consecutive steps overlap",
                "raw_bytes_per_ct": 2 * L * N * 8, "packed_bytes_per_ct": ct_bytes,
                "windows": [round(w, 1) for w in windows], "steps_per_window": e2e_steps},
        "gpu_launches": int(st1["launches"] - st0["launches"]),
        "roofline": {"kernel": "k_ks_inner (key inner product, automorphism fused)", "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": committed_traffic(),
                     "algorithmic_bytes_per_launch": alg_bytes, "rotations_per_launch": rot_per_launch,
                     "algorithmic_bytes_per_rotation": per_rot, "avg_launch_ms": round(ks_avg_ms, 5),
                     "launches_timed": ks_n,
                     "share_of_step": round(ks_ms / ms, 4)},
        "roofline_ntt": roofline_ntt,
        "roofline_bconv": roofline_bconv,
        "clocks": clk.summary(),
    }
    if extras:
        line["primitives"] = extras
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_port(args)
    ctx.close()
    del cts, ctx
    fh.api.release_memory()
    return line


# ------------------------------------------------------------------ our arm
def run_ours(args):
    """The headline: encrypted ResNet-20 (configs[3]) s/image at 128-bit security."""
    import torch
    import paper_2510_03996_b200 as fh
    from paper_2510_03996_b200 import model as M
    from paper_2510_03996_b200 import replicas

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    depth = args.depth
    spec, x = head_spec(depth)
    t_ctx = time.perf_counter()
    em = M.EncryptedModel(spec)  # 128-bit chain (model.ckks_config security=128)
    ctx = em.ctx
    ctx_s = time.perf_counter() - t_ctx
    stream = torch.cuda.ExternalStream(ctx.stream())
    xin = em.encrypt_input(x)  # the encrypted input, resident in HBM
    # batches in flight: key-sharing context clones (own stream, shared keys), one host thread each,
    # every one stepping a batch of B images in lockstep (EncryptedModel.forward_batch: bootstraps and
    # activations of the batch share their launches, keys and diagonals read once per batch)
    F = max(1, args.in_flight)
    B = max(1, args.image_batch)
    ems = [em] + [em.clone() for _ in range(F - 1)]

    def image(k):  # the seeded image first, then further seeded images of the same distribution
        return x if k == 0 else (np.random.default_rng(4100 + k).uniform(0, 1, (3, 32, 32)) - 0.5) / 0.2887

    host_images = [[image(i * B + b) for b in range(B)] for i in range(F)]
    xins = [[xin if (i == 0 and b == 0) else e.encrypt_input(host_images[i][b]) for b in range(B)]
            for i, e in enumerate(ems)]
    streams = [stream] + [torch.cuda.ExternalStream(e.ctx.stream()) for e in ems[1:]]

    def stats_all():
        tot = {}
        for e in ems:
            for k, v in e.ctx.stats().items():
                tot[k] = tot.get(k, 0) + v
        return tot

    def barrier():
        torch.cuda.synchronize()
        for e in ems:
            e.ctx.sync()
        if ws > 1:
            torch.distributed.barrier()

    # warm-up: one pass per context in turn (lazy key generation, weight plaintexts), then the
    # timed pattern itself -- all batches in flight together -- so the stream-ordered pool reaches
    # its concurrent footprint before the clock starts (mapping new pool memory mid-run costs
    # 15-20 %: measured 0.377 vs 0.318 s/image)
    for e, xi in zip(ems, xins):
        out = e.forward_batch(xi)
    out = em.forward(xin)
    del out

    # single-image latency: one stream, K steps
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0.record(stream)
    for _ in range(args.steps):
        out = em.forward(xin)
    l1.record(stream)
    l1.synchronize()
    latency_s = l0.elapsed_time(l1) / args.steps / 1e3
    del out
    barrier()

    def warm(i):  # the timed pattern, untimed (same per-batch synchronisation)
        for _ in range(max(1, args.warmup - 1)):
            ems[i].forward_batch(xins[i])
            ems[i].ctx.sync()

    th = [threading.Thread(target=warm, args=(i,)) for i in range(F)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    barrier()
    st0 = stats_all()
    prof = None
    if os.environ.get("FHEON_PROFILE_RANGE"):
        import ctypes
        prof = ctypes.CDLL("libcudart.so.12")
        prof.cudaProfilerStart()
    # throughput: F batches of B images in flight, every stream starts at e0 (stream-ordered), ends at
    # its own event
    e0 = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in ems]
    outs = [None] * F

    def run(i):
        for _ in range(args.steps):
            outs[i] = ems[i].forward_batch(xins[i])
            ems[i].ctx.sync()  # a serving loop hands each batch's result on before taking the next
        ends[i].record(streams[i])

    with ClockSampler(local) as clk:
        e0.record(stream)
        for s_ in streams[1:]:
            s_.wait_event(e0)
        h0 = time.perf_counter()
        th = [threading.Thread(target=run, args=(i,)) for i in range(F)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        host_ms = (time.perf_counter() - h0) * 1e3
        for ev in ends:
            ev.synchronize()
    ms = max(e0.elapsed_time(ev) for ev in ends)
    if prof is not None:
        prof.cudaProfilerStop()
    st1 = stats_all()
    logits_dev = outs[0][0].slots()[:em.output_count()]
    # the lockstep batch against one image at a time: same ciphertext words (image 0 of batch 0)
    single = em.forward(xin)
    batch_vs_single_words_equal = bool(np.array_equal(single.words(), outs[0][0].words()))
    del single
    out = None
    outs = None
    barrier()
    ips, ms_max = replicas.replica_throughput(ms, args.steps * F * B, torch.device("cuda", local))
    value = 1.0 / ips  # seconds per image over all ranks' images

    # ---- roofline of the dominant kernel class (NTT: integer-pipe bound), timed live in a
    # second pass of the same steps; every limb-NTT is (N/2) log2 N lazy Shoup butterflies
    n0 = ctx.stats()["ntt_limbs"]
    ctx.timer_arm(2)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    npass = max(1, min(args.steps, 3))
    f0.record(stream)
    for _ in range(npass):
        out = em.forward_batch(xins[0])  # the timed region's unit of work: one lockstep batch
    f1.record(stream)
    f1.synchronize()
    pass_ms = f0.elapsed_time(f1)
    ntt_ms, ntt_n = ctx.timer_read()
    ctx.timer_arm(0)
    del out
    ntt_limbs = ctx.stats()["ntt_limbs"] - n0
    bfly = ntt_limbs * (N // 2) * LOGN
    try:
        bpeak = json.load(open(os.path.join(ROOT, "profiles", "int_peak.json")))["shoup_ct_butterflies_per_s"]
        bsrc = "measured (profiles/int_peak.json: lazy Shoup butterfly, IMAD.WIDE-bound, all 148 SMs)"
    except Exception:
        bpeak, bsrc = 8.7e11, "fallback"
    ntt_rate = bfly / (ntt_ms / 1e3)
    roofline = {"kernel": "ntt_phase_kernel (COL + ROW phases, forward + inverse; every limb-NTT of the step)",
                "bound": "int", "achieved": round(ntt_rate / 1e9, 1), "peak": round(bpeak / 1e9, 1),
                "unit": "Gbutterfly/s", "frac": round(ntt_rate / bpeak, 4), "peak_source": bsrc,
                "algorithmic_work": "(N/2) log2 N = 524288 butterflies per 2^16 limb-NTT",
                "limb_ntts_per_image": ntt_limbs // (npass * B), "launch_scopes_timed": ntt_n,
                "measured_on": f"one lockstep batch of {B} images on one stream (the unit each of the "
                               f"{F} in-flight streams runs in the timed region)",
                "avg_scope_ms": round(ntt_ms / max(1, ntt_n), 5),
                "share_of_step": round(ntt_ms / pass_ms, 4),
                "hbm_gbs": round(ntt_limbs * N * 8 * 4 / (ntt_ms / 1e3) / 1e9, 1),
                "traffic": None,
                "traffic_note": "profiles/r02_ncu_resnet_ntt.csv"}
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        roofline["traffic"] = tr["resnet_ntt_mean_dram_bytes_per_launch"]
        roofline["algorithmic_bytes_per_launch"] = tr["resnet_ntt_mean_algorithmic_bytes_per_launch"]
        roofline["traffic_note"] = ("mean DRAM bytes per NTT phase launch, ncu --set full of 32 launches of a "
                                    "one-image step (profiles/r02_ncu_resnet_ntt.csv): 0.72 of the "
                                    "algorithmic 16 N bytes per limb -- integer-bound, no wasted re-reads")
    except Exception:
        pass

    # ---- e2e through the public API: host images -> encode + encrypt -> forward -> decrypt -> host
    # logits, the same F batches of B in flight (EncryptedModel.infer_batch from F host threads);
    # wall clock from the first call to the last result on the host
    e2e_steps = max(3, args.steps // 2)
    e2e_out = [None] * F

    def run_e2e(i, n):
        for _ in range(n):
            e2e_out[i] = ems[i].infer_batch(host_images[i])

    def e2e_pass(n):
        th = [threading.Thread(target=run_e2e, args=(i, n)) for i in range(F)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    e2e_pass(1)
    barrier()
    t0 = time.perf_counter()
    e2e_pass(e2e_steps)
    barrier()
    e2e_ips, _ = replicas.replica_throughput((time.perf_counter() - t0) * 1e3, e2e_steps * F * B,
                                             torch.device("cuda", local))
    logit_err_dev_vs_api = float(np.abs(e2e_out[0][0] - logits_dev).max())
    # one image at a time through infer() (latency shape of the same path)
    t0 = time.perf_counter()
    for _ in range(3):
        r = em.infer(x)
    e2e_latency_s = (time.perf_counter() - t0) / 3
    del r

    line = {
        "metric": "encrypted inference s/image (ResNet-20, CKKS N=2^16, full bootstrapping, 128-bit security)",
        "value": round(value, 4),
        "unit": "s/image",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max / args.steps, 3),
        "host_enqueue_ms_per_step": round(host_ms / args.steps, 3),
        "images_in_flight": F * B,
        "batches_in_flight": F,
        "batch": B,
        "latency_s_per_image": round(latency_s, 4),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64 (RNS limbs, <=61-bit primes; int8 tensor-core basis conversion)",
        "data": "synthetic (seeded input and He-normal weights; no CIFAR-10 / trained weights in the container)",
        "config": dict(head_config(depth), parallelism=f"replicas x{ws}"),
        "security": em.security,
        "chain": {"limbs": ctx.L, "special_limbs": ctx.K, "dnum": ctx.dnum, "bootstraps": em.n_boot,
                  "context_create_s": round(ctx_s, 2), "key_bytes": ctx.key_bytes()},
        "e2e": {"value": round(1.0 / e2e_ips, 4), "unit": "s/image",
                "h2d_bytes_per_step": N * 8 * F * B, "d2h_bytes_per_step": 2 * N * 8 * F * B,
                "path": "EncryptedModel.infer_batch (public API) from F host threads: host images -> "
                        "h2d of the slot values -> device special-FFT encode + RNS + NTT + encrypt -> "
                        "forward_batch -> device decrypt -> d2h of 2 limbs per image -> host CRT + decode -> "
                        "logits on the host",
                "steps": e2e_steps, "logits_max_abs_diff_vs_value_path": logit_err_dev_vs_api,
                "images_in_flight": F * B, "latency_s_per_image": round(e2e_latency_s, 4)},
        "value_note": f"{F} batches of {B} images in flight per GPU: key-sharing context clones "
                      f"(SlotContext.clone, one stream and host thread each), each stepping its batch in "
                      f"lockstep (forward_batch: bootstraps / activations of the batch share launches, keys "
                      f"and diagonals); latency_s_per_image is one image at a time; a batched image's "
                      f"ciphertext words equal the one-at-a-time result: {batch_vs_single_words_equal}",
        "gpu_launches": int(st1["launches"] - st0["launches"]),
        "ops_per_image": {k: int((st1[k] - st0[k]) // (args.steps * F * B)) for k in
                          ("rotations", "keyswitches", "mult_plain", "mult_cipher", "rescales", "ntt_limbs")},
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    for e in ems:  # the keys (~31 GB) must not outlive the headline: the model cases need the HBM
        e.ctx.close()
    del em, ems, ctx, xin, xins, streams
    fh.api.release_memory()
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_reference(spec, x, depth)
        line["logits_max_abs_err_vs_reference"] = line["cpu_baseline"].pop("_logit_err_fn")(logits_dev)
    if not args.quick and not args.no_rotations:
        rot = rotation_bench(args)
        if rank == 0:
            line["rotations"] = rot
    if rank == 0 and not args.quick and not args.no_models:
        line["models"] = model_runs(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def host_cpu():
    """The GPU box's host: lscpu model name and logical core count."""
    model = None
    try:
        for ln in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def reference_config1_conv():
    """BASELINE configs[0] through the reference's own convolution() (layers_conv.cpp:577-594,
    oracle/_ref) on this host, same seeded input / weights as our config-1 layer: mean of 50."""
    from oracle import ref as sref
    r = sref.Ref(16384, 8192, 10)
    x = np.random.default_rng(1001).uniform(0, 1, (1, 28, 28))
    w = np.random.default_rng(1002).normal(0, 0.1, (6, 1, 5, 5))
    r.convolution(x, 10, 1, 28, 6, 5, 1, 0, 0, 0, w, None)
    t0 = time.perf_counter()
    for _ in range(50):
        r.convolution(x, 10, 1, 28, 6, 5, 1, 0, 0, 0, w, None)
    return round((time.perf_counter() - t0) / 50 * 1e3, 3)


def cpu_baseline_reference(spec, x, depth):
    """The reference's own infer() (oracle/_ref, the unmodified slotcnn core) on the
    same spec, weights and input: one image on one host core."""
    import tempfile
    from oracle import ref as sref
    if not sref.available():
        return {"value": None, "unit": "s/image", "cores": 1, "kind": "reference",
                "sample": "oracle/_ref not built", "_logit_err_fn": lambda lg: None}
    path = spec.write(tempfile.mkdtemp())
    sref.infer(path, x)  # warm (page-in)
    t0 = time.perf_counter()
    rl, rows, _, rwall = sref.infer(path, x)
    dt = time.perf_counter() - t0
    return {"value": round(dt, 4), "unit": "s/image", "cores": 1, "kind": "reference",
            "sample": f"one ResNet-20 image through the reference's infer() (slotcnn cleartext slot simulator, "
                      f"N=2^16 depth {depth}, {sum(1 for r in rows if r[3])} top-level bootstraps)",
            "reference_internal_wall_s": round(rwall / 1e3, 4), "host": host_cpu(),
            "reference_config1_conv_ms_1core": reference_config1_conv(),
            "_logit_err_fn": lambda lg: float(np.abs(np.asarray(lg)[:rl.size] - rl).max())}


def primitives(ctx, fh):
    """Config-2 microbench (device time, CUDA events) + config-1 conv layer."""
    out = {}
    kinds = {"ntt_ms_per_ct": 0, "intt_ms_per_ct": 1, "automorphism_ms_per_ct": 2, "rotation_ms": 3,
             "mac_term_ms_per_ct": 5, "rescale_ms_per_ct": 6, "add_ms_per_ct": 7}
    for name, k in kinds.items():
        batch = 1 if k == 3 else 8
        ms = ctx.microbench(k, batch, L, 1, 10)
        out[name] = round(ms / batch, 5)
    for r in (8, 32):
        ms = ctx.microbench(4, 1, L, r, 5)
        out[f"hoisted{r}_rot_per_s"] = round(r / (ms / 1e3), 1)
    ntt_bytes = 2 * L * N * 8 * 2
    out["ntt_hbm_gbs"] = round(ntt_bytes / (out["ntt_ms_per_ct"] / 1e3) / 1e9, 1)
    # ---- the SURVEY 8(d) C2 sweep
    peak, _ = measured_peak_hbm()
    alpha = (L + DNUM - 1) // DNUM
    beta = (L + alpha - 1) // alpha
    key_bytes = 16 * beta * (L + K) * N
    sweep = {}
    for B in (1, 2, 4, 8, 16, 32, 64):  # same key across B ciphertexts: one key read per launch
        ms = ctx.microbench(8, B, L, 1, 5)
        alg = B * 32 * L * N + key_bytes  # B 32 l N + 16 beta (l + K) N
        sweep[str(B)] = {"rot_per_s": round(B / (ms / 1e3), 1), "ms": round(ms, 4),
                         "hbm_frac_of_algorithmic": round(alg / (ms / 1e3) / 1e9 / peak, 4)}
    out["same_key_batched_rotation"] = {
        "by_batch": sweep, "hbm_roofline_rot_per_s_at_64": round(64 / ((64 * 32 * L * N + key_bytes) / (peak * 1e9)), 1),
        "note": "rot/s of B distinct ciphertexts rotated by one step; roofline = algorithmic bytes "
                "B 32 l N + 16 beta (l + K) N at the measured HBM peak (SURVEY 8(d))"}
    out["mac_fused_ms"] = {str(k): round(ctx.microbench(9, 1, L, k, 10), 5) for k in (1, 9, 25)}
    out["mac_fused_hbm_frac"] = {k: round((int(k) * 24 * L * N + 16 * L * N) / (v / 1e3) / 1e9 / peak, 4)
                                 for k, v in out["mac_fused_ms"].items()}
    n_auto = S - 1
    ms_all = ctx.microbench(10, 1, L, 1, n_auto)  # every t in [1, S), one launch each
    out["automorphism_all_steps"] = {"steps": n_auto, "mean_ms": round(ms_all, 5),
                                     "hbm_gbs": round(2 * 2 * L * N * 8 / (ms_all / 1e3) / 1e9, 1)}
    # integer roofline of the NTT: (N/2) log2 N butterflies per limb-poly, 2L limb-polys
    bfly = (N // 2) * LOGN * 2 * L
    achieved = bfly / (out["ntt_ms_per_ct"] / 1e3)
    try:
        peak = json.load(open(os.path.join(ROOT, "profiles", "int_peak.json")))["shoup_ct_butterflies_per_s"]
        src = "measured (profiles/int_peak.json: lazy Shoup butterfly, IMAD.WIDE-bound)"
    except Exception:
        peak, src = 8.7e11, "fallback"
    out["ntt_int_roofline"] = {"bound": "int", "achieved": round(achieved / 1e9, 1), "peak": round(peak / 1e9, 1),
                               "unit": "Gbutterfly/s", "frac": round(achieved / peak, 4), "peak_source": src,
                               "butterflies_per_ct": bfly}
    # config-1 conv layer (BASELINE configs[0]) through the layer API
    try:
        c1 = fh.SlotContext(fh.ContextConfig.preset("config1"))
        rng = np.random.default_rng(1001)
        x = rng.uniform(0, 1, (1, 28, 28))
        w = np.random.default_rng(1002).normal(0, 0.1, (6, 1, 5, 5))
        cfg = fh.ConvConfig(1, 6, 5, 1, 0)
        xs = fh.SlotVector.encode(c1, x.reshape(-1))
        fh.convolution(fh.PackedTensor(xs, 1, 28), cfg, fh.KernelTensor(w))  # warm + keygen
        c1.sync()
        t0 = time.perf_counter()
        reps = 5
        for _ in range(reps):
            r = fh.convolution(fh.PackedTensor(xs, 1, 28), cfg, fh.KernelTensor(w))
        c1.sync()
        out["config1_conv_layer_ms"] = round((time.perf_counter() - t0) / reps * 1e3, 3)
        del r
    except Exception as e:  # pragma: no cover - diagnostics only
        out["config1_conv_layer_error"] = str(e)
    return out


def model_cases(args, want=None):
    """The model cases of the bench: (name, spec, input, security, reference-schedule-only).
    Encrypted inference s/image of the other BASELINE networks and chains through the
    model runtime (host image -> encrypt -> every layer and bootstrap on the GPU ->
    decrypt), with the decrypted logits compared against the reference's own infer()
    on the same spec / weights / input (timed beside it on one core) and the chain's
    security disclosure.  Chains that cannot reach 128 bits (the reference's presets:
    depth 25 at N = 2^14 / 2^15; LeNet-5 at configs[2]'s N = 2^15, where bootstrapping
    alone needs more modulus than the 881-bit bound) run with security=0 and say so.
    want: build only that case (the others are returned as names with None)."""
    import tempfile
    from paper_2510_03996_b200 import model as M
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from model_files import materialize

    def norm(x):
        return (x - 0.5) / 0.2887

    def lenet_ref():
        spec = M.load_spec(materialize("lenet5", tempfile.mkdtemp(), seed=9))
        spec = M.calibrate_relu_scales(spec, [np.random.default_rng(500 + i).uniform(0, 1, (1, 28, 28))
                                              for i in range(4)])
        return spec, np.random.default_rng(501).uniform(0, 1, (1, 28, 28))

    def resnet_cal():
        return [norm(np.random.default_rng(4002 + i).uniform(0, 1, (3, 32, 32))) for i in range(6)]

    xl = np.random.default_rng(3001).uniform(0, 1, (1, 28, 28))
    builders = [("lenet5_configs2_n15_d25", lambda: (M.lenet5(ring=32768, depth_budget=25), xl), 0, False),
                ("lenet5_n16_d10_128bit", lambda: (M.lenet5(ring=65536, depth_budget=10), xl), 128, False),
                ("lenet5_reference_spec", lenet_ref, 0, False)]
    if not args.no_resnet:
        if not args.no_reference_schedule:
            builders.append((f"resnet20_n16_d{args.depth}_128bit_reference_schedule", lambda: head_spec(args.depth),
                             128, True))
        builders.append(("resnet20_reference_spec", lambda: (M.calibrate_relu_scales(
            M.load_spec(materialize("resnet20", tempfile.mkdtemp(), seed=9)), resnet_cal()), head_spec(args.depth)[1]),
            0, False))
        builders.append(("resnet20_n16_d25_insecure", lambda: (M.calibrate_relu_scales(
            M.resnet20(ring=65536, depth_budget=25), resnet_cal()), head_spec(args.depth)[1]), 0, False))
        if not args.no_vgg:
            builders.append(("vgg16_paper_widths_n16_128bit", lambda: (M.calibrate_relu_scales(
                M.vgg16_paper(ring=65536, depth_budget=args.depth),
                [norm(np.random.default_rng(5002 + i).uniform(0, 1, (3, 32, 32))) for i in range(4)]),
                norm(np.random.default_rng(5001).uniform(0, 1, (3, 32, 32)))), 128, False))
    cases = []
    for name, build_fn, security, ref_only in builders:
        if want is not None and name != want:
            cases.append((name, None, None, security, ref_only))
            continue
        spec, x = build_fn()
        cases.append((name, spec, x, security, ref_only))
    return cases


def run_model_case(args, case):
    """One model case (built by model_cases) timed in THIS process: encrypted s/image with
    clocks sampled, the logit error against the reference's infer(), key residency."""
    import tempfile
    import paper_2510_03996_b200 as fh
    from paper_2510_03996_b200 import model as M
    try:
        from oracle import ref as sref
        have_ref = sref.available()
    except Exception:
        have_ref = False
    name, spec, x, security, ref_schedule_only = case
    em = M.EncryptedModel(spec, security=security, schedule="reference" if ref_schedule_only else "fast")
    reps = 1 if ref_schedule_only else args.model_reps
    for _ in range(1 if ref_schedule_only else 3):  # warm-up: lazy keys, plaintext caches, pool growth
        em.infer(x)
    times = []
    with ClockSampler(0) as clk:
        for _ in range(reps):
            r = em.infer(x)
            times.append(r.wall_ms / 1e3)
    rec = {"s_per_image": round(float(np.median(times)), 4), "reps": reps,
           "schedule": "reference (the reference's exact rotation sequence)" if ref_schedule_only else "fast",
           "rep_times_s": [round(t, 4) for t in times],
           "spec": ("the reference's models/%s.json (preset, seeded weights)" % name.split("_")[0]
                    if name.endswith("reference_spec") else "paper_2510_03996_b200.model." + name.split("_")[0]),
           "ring_dimension": spec.ring_dimension, "depth_budget": spec.depth_budget, "security": em.security,
           "limbs": em.ctx.L, "special_limbs": em.ctx.K, "dnum": em.ctx.dnum, "bootstraps": em.n_boot,
           "rotations": r.stats["rotations"], "keyswitches": r.stats["keyswitches"],
           "gpu_launches": r.stats["launches"], "key_bytes": em.ctx.key_bytes(), "clocks": clk.summary(),
           "data": "synthetic seeded input, seeded random weights (no datasets/weights in the container)"}
    if name == "resnet20_reference_spec":
        # keyplan block mode (model_run.cpp:150 key_mode): keys of one block resident at a time
        preload_key_bytes = em.ctx.key_bytes()
        em.infer(x, key_mode="block")
        rb = em.infer(x, key_mode="block", verify_keys=True)
        est = M.keyplan.estimate_memory(rb.plan, em.memory_model())
        ref_est = M.keyplan.estimate_memory(rb.plan, M.keyplan.MemoryModel.reference_model(
            spec.ring_dimension, spec.depth_budget, 3))
        # the same plan with the keys streamed from pinned host memory (packed wire format,
        # upload stream) instead of regenerated: the PCIe key traffic is inside s/image
        em.enable_key_streaming()
        em.infer(x, key_mode="block")
        rs = em.infer(x, key_mode="block", verify_keys=True)
        rec["key_mode_block_streamed"] = {
            "s_per_image": round(rs.wall_ms / 1e3, 4), "keys_uploaded_per_image": rs.key_residency["uploaded"],
            "key_bytes_uploaded_per_image": rs.key_residency["uploaded_bytes"],
            "keys_generated_per_image": rs.key_residency["generated"], "trace_check_ok": rs.trace_check.ok(),
            "pcie_gbs_implied": round(rs.key_residency["uploaded_bytes"] / (rs.wall_ms / 1e3) / 1e9, 2)}
        rec["key_mode_block"] = {
            "s_per_image": round(rb.wall_ms / 1e3, 4), "blocks": len(rb.plan.blocks),
            "trace_check_ok": rb.trace_check.ok(), "rotations_checked": rb.trace_check.rotations_checked,
            "keys_generated_per_image": rb.key_residency["generated"],
            "peak_key_bytes": rb.key_residency["peak_key_bytes"], "preload_key_bytes": preload_key_bytes,
            "estimate": {"total_keys": est.total_keys, "peak_resident_keys": est.resident_keys,
                         "preload_bytes": est.preload_bytes, "peak_bytes": est.peak_bytes,
                         "reference_memory_model_preload_bytes": ref_est.preload_bytes}}
    if have_ref:
        path = spec.write(tempfile.mkdtemp())
        rl, rows, _, rwall = sref.infer(path, x)
        rec["max_abs_logit_err_vs_reference"] = float(np.abs(r.logits - rl).max())
        rec["argmax_match"] = bool(int(np.argmax(r.logits)) == int(np.argmax(rl)))
        rec["reference_sim_s_per_image_1core"] = round(rwall / 1e3, 4)
    del em
    return rec


def model_runs(args):
    """Every model case in a FRESH process (`bench.py --model-case NAME`): each starts from
    an empty device and pool, as a deployment running that model would -- one
    process's earlier workloads measurably slowed later ones (VGG-16 0.70 s alone,
    1.1 s after the headline section in the same process)."""
    out = {}
    try:
        import torch
        free, total = torch.cuda.mem_get_info()
        out["_parent_device_memory_free_gb"] = round(free / 1e9, 1)
    except Exception:
        pass
    names = [c[0] for c in model_cases(args, want="")]
    only = [c for c in (args.models or "").split(",") if c]
    for name in names:
        if only and not any(name.startswith(c) for c in only):
            continue
        cmd = [sys.executable, os.path.abspath(__file__), "--model-case", name, "--depth", str(args.depth),
               "--model-reps", str(args.model_reps)]
        if args.no_reference_schedule:
            cmd.append("--no-reference-schedule")
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        try:
            out[name] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            out[name] = {"error": (r.stderr or r.stdout)[-800:]}
    return out


def cpu_baseline_port(args):
    """The repo's CPU RNS-CKKS oracle doing config-2 rotations (OpenMP over limbs)."""
    from oracle.ckks_oracle import Oracle
    o = Oracle(LOGN, L, K, DNUM, 60, 50, 60, 1)
    rng = np.random.default_rng(2001)
    ct = o.encrypt(rng.uniform(-1, 1, S), 0)
    keys = [o.rotation_key(1 << i) for i in range(2)]
    o.rotate(ct, 1, keys[0])  # warm
    n = args.cpu_sample
    t0 = time.perf_counter()
    for i in range(n):
        o.rotate(ct, 1 << (i % 2), keys[i % 2])
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": round(n / dt, 3), "unit": "rotations/s", "cores": cores, "kind": "port",
            "sample": f"{n} key-switch rotations at N=2^16, L=24, dnum=3 (oracle/ckks_oracle.c, OpenMP)"}


# ------------------------------------------------------------ reference arm
def run_reference(args):
    """The reference's own CPU path for the headline: its infer()
    (model_run.cpp:100-159, oracle/_ref = the unmodified slotcnn core) on the same
    spec, weights and input as our arm.  value = 1-thread latency (median over
    the steps); all-core throughput with one inference per host thread beside it."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import tempfile
    from oracle import ref as sref
    if not sref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libslotcnn_ref.so not built"}))
        return
    depth = args.depth
    spec, x = head_spec(depth)
    path = spec.write(tempfile.mkdtemp())
    for _ in range(args.warmup):
        sref.infer(path, x)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, rows, _, _ = sref.infer(path, x)
        times.append(time.perf_counter() - t0)
    value = float(np.median(times))
    cores = os.cpu_count() or 1
    res = [None] * cores

    def work(i):
        res[i] = sref.infer(path, x)

    th = [threading.Thread(target=work, args=(i,)) for i in range(cores)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    par = time.perf_counter() - t0
    line = {
        "impl": "reference",
        "metric": "encrypted inference s/image (ResNet-20, CKKS N=2^16, full bootstrapping, 128-bit security)",
        "value": round(value, 4),
        "unit": "s/image",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(value * 1e3, 3),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 (cleartext slot simulator)",
        "data": "synthetic (seeded input and He-normal weights)",
        "config": dict(head_config(depth), parallelism=f"replicas x{ws}"),
        "cpu_baseline": {"value": round(value, 4), "unit": "s/image", "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} single-thread infer() calls of the reference (oracle/_ref) on the "
                                   f"headline spec, median; {sum(1 for r in rows if r[3])} top-level bootstraps"},
        "e2e": {"value": round(value, 4), "unit": "s/image", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "all_core_throughput": {"images": cores, "threads": cores, "wall_s": round(par, 3),
                                "s_per_image": round(par / cores, 4)},
        "host": host_cpu(),
        "reference_config1_conv_ms_1core": reference_config1_conv(),
        "rep_times_s": [round(t, 4) for t in times],
        "note": "the reference's backend is a cleartext slot simulator (backend.cpp:165-249: rotate is a memcpy, "
                "bootstrap a level reset) -- it does no cryptography; the paper's OpenFHE CPU figure for "
                "ResNet-20 is 403 s/image (BASELINE.md)",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--cpu-sample", type=int, default=12)
    ap.add_argument("--ref-iters", type=int, default=2000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quick", action="store_true", help="skip the primitive breakdown and the models")
    ap.add_argument("--no-models", action="store_true", help="skip LeNet-5 / ResNet-20 s/image")
    ap.add_argument("--no-resnet", action="store_true", help="skip the ResNet-20 / VGG-16 model variants")
    ap.add_argument("--no-vgg", action="store_true", help="skip VGG-16")
    ap.add_argument("--depth", type=int, default=HEAD_DEPTH, help="ResNet-20 depth budget of the headline chain")
    ap.add_argument("--in-flight", type=int, default=3,
                    help="batches in flight per GPU (key-sharing contexts, one host thread each)")
    ap.add_argument("--image-batch", type=int, default=3, help="images per lockstep batch (forward_batch)")
    ap.add_argument("--models", default="", help="comma-separated name prefixes of the model cases to run")
    ap.add_argument("--no-rotations", action="store_true", help="skip the configs[1] rotation block")
    ap.add_argument("--model-case", default="", help=argparse.SUPPRESS)
    ap.add_argument("--model-reps", type=int, default=3)
    ap.add_argument("--no-reference-schedule", action="store_true",
                    help="skip the models' reference-rotation-schedule timing")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.model_case:
        case = [c for c in model_cases(args, want=args.model_case) if c[0] == args.model_case]
        if not case:
            raise SystemExit(f"unknown model case {args.model_case}")
        print(json.dumps(run_model_case(args, case[0])), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
