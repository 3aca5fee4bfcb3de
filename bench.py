#!/usr/bin/env python3
"""Benchmark of the FSDP2 Shard(0) hot path (BASELINE.json metric: "FSDP unshard+reshard
GB/s per layer (fraction of NVLink/HBM peak) at 1/2/4/8 B200").

One step = one pass of the whole hot path over the Llama 3.1 8B parameter layout
(BASELINE.json configs[1]): for every FSDP unit (32 TransformerBlocks + root)
unshard (bf16; W=1: one cast kernel into the unsharded tensors, W>1: the fused NVLink push
kernel, or copy-in -> NCCL all-gather -> copy-out with --algo nccl) -> reshard ->
reduce_scatter_grads (fp32 reduction with one /W: W=1 the RS copy-in kernel, W>1 the fused
store-scatter + local reduce or pull kernels, or chunk-cat -> NCCL reduce-scatter), with the
next unit's unshard prefetched.  Bytes per unit: the all-gather
output W*S*2 plus the reduce-scatter input W*S*4 per rank; `value` = those bytes summed
over all ranks / max-over-ranks step time (whole job, weak scaling: every rank unshards
the full model).

Launch: python bench.py [--gpus N --steps K --warmup W]; for N > 1 under torchrun.
`--impl reference` times the CPU oracle (the reference arm of this tier) instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "llama3.1-8b": dict(model="llama3.1-8b", fp8=False, cycle=None),
    "llama3.1-8b-fp8": dict(model="llama3.1-8b", fp8=True, cycle=None),
    "llama3.1-70b": dict(model="llama3.1-70b", fp8=False, cycle=4),
    "toy": dict(model="toy", fp8=False, cycle=None),
}
METRIC = "FSDP unshard+reshard GB/s per layer (fraction of NVLink/HBM peak)"
NVLINK_GBS = 900.0          # NVLink 5 per direction per GPU, nominal (BASELINE.json north_star)
NVLINK_MEASURED_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
HBM_NOMINAL_GBS = 8000.0     # "~8 TB/s" (BASELINE.json north_star)


def wire_report(wire_rank, ms, ms_iso, W, R, hsdp_wp=False):
    """Physical NVLink bytes per rank per direction per step / step time, vs 900 and 770."""
    if not wire_rank:
        return None
    g = wire_rank / (ms * 1e-3) / 1e9
    gi = wire_rank / (ms_iso * 1e-3) / 1e9
    return {"bytes_per_step_per_rank_per_direction": int(wire_rank),
            "GBps_per_direction": round(g, 1), "frac_of_900": round(g / NVLINK_GBS, 4),
            "frac_of_770": round(g / NVLINK_MEASURED_GBS, 4),
            "isolated_GBps_per_direction": round(gi, 1), "isolated_frac_of_900": round(gi / NVLINK_GBS, 4),
            "isolated_frac_of_770": round(gi / NVLINK_MEASURED_GBS, 4),
            "model": "P2P: (W-1) x own cast rows (push) + (W-1) x own bf16 grad rows (reduce-scatter); "
                     "NCCL ring: (W-1) x slot + (W-1) x 4S" + (
                         "; HSDP world RS: (R W - 1) x own bf16 grad rows (two-phase: / R, + (R-1) fp32 pieces "
                         "of own / R) instead of the shard-group RS"
                         if hsdp_wp else ("; + fp32 replica all-reduce" if R > 1 else ""))}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)   # >= 30 steps and >= 0.5 s
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama3.1-8b", choices=list(WORKLOADS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--serial", action="store_true", help="no prefetch: each unit isolated")
    ap.add_argument("--algo", default="auto", choices=["auto", "nccl", "p2p"],
                    help="collectives: fused NVLink peer-memory kernels (p2p) or NCCL; auto = library default")
    ap.add_argument("--step", default="unit", choices=["unit", "train"],
                    help="unit: every FSDP unit once through unshard -> reshard -> reduce-scatter; "
                         "train: the paper's training-step pattern (forward unshards with prefetch, the last "
                         "block kept unsharded, backward re-unshards in reverse + reduce-scatter, P:424-431)")
    ap.add_argument("--zero2", action="store_true",
                    help="with --step train: reshard_after_forward=False for every block (ZeRO-2, P:636)")
    ap.add_argument("--shard-size", type=int, default=0, help="HSDP: data_parallel_shard_degree (default all ranks)")
    ap.add_argument("--p2p-rs", default="auto", choices=["auto", "store", "pull"],
                    help="P2P reduce-scatter mechanism: peers store rows into owners' receive buffers, or owners "
                         "pull rows from peers' staging (auto = library default)")
    ap.add_argument("--grads", default="auto", choices=["auto", "torch", "library"],
                    help="where the full grads live: torch tensors (the RS stages them), or the layer's "
                         "own symmetric grad buffers (zero-copy; auto = library under P2P)")
    ap.add_argument("--compute-tokens", type=int, default=0,
                    help="optional compute proxy (SURVEY.md 8(d) row 4; bf16 unit step only): after each unit's "
                         "wait_unshard, bf16 GEMMs x[T, in] @ W_p^T over its gathered 2-D weights, 3 passes "
                         "(6*N*T flops, forward + backward), so prefetch/RS overlap with compute is measured; "
                         "also times the compute alone -> exposed communication")
    ap.add_argument("--graph", action="store_true",
                    help="capture the step into a CUDA graph after the warm-up and time its replays (for "
                         "launch-bound units, e.g. --workload toy); kernel statistics then come from one eager "
                         "profiled step")
    ap.add_argument("--fp8-scaling", default="dynamic", choices=["dynamic", "delayed"],
                    help="float8 workloads: dynamic (amax pass over every shard each step) or delayed "
                         "(history of 16; the amax is fused into the fp8 unshard's cast, P:157)")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def unit_lists(model: str, include_root=True):
    import synth
    units = synth.model_units(model, include_root=include_root)
    return [([s for _, s, _ in u], [e for _, _, e in u]) for u in units]


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", ",".join(str(g) for g in self.gpus)],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.06)   # one more sample interval; more would add idle samples to the median
        self.proc.terminate()
        self.proc.wait(timeout=10)
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2410_06511_b200 as F

    N = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if N != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={N}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
        mesh = F.Mesh.from_process_group(device=local, shard_size=args.shard_size or None)
    else:
        mesh = F.Mesh(1, 0, local, unique_id=F.get_unique_id())
    if args.algo != "auto" and N > 1:
        mesh.set_algo(args.algo)
    if args.p2p_rs != "auto" and N > 1:
        mesh.set_p2p_rs(args.p2p_rs)
    algo = mesh.algo if N > 1 else "local (W=1: identity collectives)"
    if N > 1 and mesh.algo == "p2p":
        algo += f" (reduce-scatter: {mesh.p2p_rs})"
    hsdp_mode = mesh.hsdp_rs if N > 1 and mesh.replicate_size > 1 else None
    hsdp_wp = hsdp_mode in ("world_pull", "world_pull_2phase")
    hsdp_2ph = hsdp_mode == "world_pull_2phase"
    if hsdp_mode:
        algo += f"; HSDP {mesh.replicate_size}x{mesh.shard_size} reduce-scatter: " + {
            "world_pull_2phase": "two-phase world RS (1/R pieces over all ranks + replica gather, nested order)",
            "world_pull": "world pull (one kernel over all ranks, nested order)"}.get(hsdp_mode,
                                                                                    "shard-group RS + NCCL all-reduce")
    wl = WORKLOADS[args.workload]
    units = unit_lists(wl["model"])
    if wl["cycle"]:   # 70B: cycle `cycle` distinct block instances (memory), SURVEY.md §8(d) row 4
        units = units[:wl["cycle"]]
    pdtype = torch.float8_e4m3fn if wl["fp8"] else torch.bfloat16

    # ---- setup: shard (synthetic seeded params written straight into the shards)
    layers, grads = [], []
    gen = torch.Generator(device=dev).manual_seed(241006511 + rank)
    lib_grads = args.grads == "library" or (args.grads == "auto" and N > 1 and (
        hsdp_wp or (mesh.algo == "p2p" and mesh.p2p_rs != "store")))   # store mode reads any grads
    for ui, (shapes, elig) in enumerate(units):
        l = F.fsdp_shard(mesh, None, elig, shapes=shapes)
        flat = l.sharded_flat()
        for p in range(l.P):
            m = l.metas[p]
            n = m["row_count"] * m["rest"]
            if n:
                flat[m["elem_offset"]:m["elem_offset"] + n].normal_(0.0, 0.02, generator=gen)
        layers.append(l)
        g = [(torch.randn(s, generator=gen, device=dev) * 1e-3).to(torch.bfloat16) for s in shapes]
        if lib_grads:   # the backward would write its grads straight into the layer's buffer
            bufs = l.full_grad_buffers(torch.bfloat16)
            for b, x in zip(bufs, g):
                b.copy_(x)
            g = bufs
        grads.append(g)
    torch.cuda.synchronize()
    comp = torch.cuda.Stream(device=dev)
    W = mesh.shard_size if N > 1 else 1     # Shard(0) degree (HSDP: shard group size)

    T = args.compute_tokens
    if T and (wl["fp8"] or args.step != "unit"):
        raise SystemExit("--compute-tokens: bf16 workloads with --step unit only")
    xin = {}
    if T:
        for l in layers:
            for s in l.shapes:
                if len(s) == 2 and s[1] not in xin:
                    xin[s[1]] = torch.randn(T, s[1], generator=gen, device=dev).to(torch.bfloat16)

    def compute(weights):
        """3 forward-shaped GEMM passes over the unit's 2-D weights (6*N*T flops)."""
        with torch.cuda.stream(comp):
            for _ in range(3):
                for w in weights:
                    if w.dim() == 2:
                        torch.matmul(xin[w.shape[1]], w.t())

    def step_unit():
        n = len(layers)
        if not args.serial:
            F.fsdp_unshard(layers[0], pdtype, stream=comp)
        for i in range(n):
            if args.serial:
                F.fsdp_unshard(layers[i], pdtype, stream=comp)
            F.fsdp_wait_unshard(layers[i], stream=comp)
            if not args.serial and i + 1 < n:
                F.fsdp_unshard(layers[i + 1], pdtype, stream=comp)   # prefetch
            if T:
                compute(layers[i].unsharded_params())
            F.fsdp_reshard(layers[i], stream=comp)
            F.reduce_scatter_grads(layers[i], grads[i], stream=comp)
            if args.serial:
                F.fsdp_wait_reduce_scatter(layers[i], stream=comp)
        for l in layers:
            F.fsdp_wait_reduce_scatter(l, stream=comp)

    # --step train: root (last unit) wraps the blocks; forward unshards root then
    # every block with the next prefetched, reshards each block after use except the last
    # — or none under ZeRO-2 — and keeps the root unsharded through the
    # forward; backward re-unshards what was resharded in reverse order (prefetching the
    # previous block), reduce-scatters each block's grads and finally the root's.
    blocks, root = layers[:-1], layers[-1]
    kept = set(range(len(blocks))) if args.zero2 else {len(blocks) - 1}

    def step_train():
        F.fsdp_unshard(root, pdtype, stream=comp)
        F.fsdp_wait_unshard(root, stream=comp)
        F.fsdp_unshard(blocks[0], pdtype, stream=comp)
        for i, b in enumerate(blocks):                      # forward
            F.fsdp_wait_unshard(b, stream=comp)
            if i + 1 < len(blocks):
                F.fsdp_unshard(blocks[i + 1], pdtype, stream=comp)
            if i not in kept:
                F.fsdp_reshard(b, stream=comp)
        F.fsdp_reshard(root, stream=comp)
        F.fsdp_unshard(root, pdtype, stream=comp)            # backward: output layer first
        F.fsdp_wait_unshard(root, stream=comp)
        order = list(range(len(blocks)))[::-1]
        if order[0] not in kept:
            F.fsdp_unshard(blocks[order[0]], pdtype, stream=comp)
        for j, i in enumerate(order):
            b = blocks[i]
            F.fsdp_wait_unshard(b, stream=comp)
            if j + 1 < len(order) and order[j + 1] not in kept:
                F.fsdp_unshard(blocks[order[j + 1]], pdtype, stream=comp)   # backward prefetch
            F.fsdp_reshard(b, stream=comp)
            F.reduce_scatter_grads(b, grads[i], stream=comp)
        F.fsdp_reshard(root, stream=comp)
        F.reduce_scatter_grads(root, grads[-1], stream=comp)
        for l in layers:
            F.fsdp_wait_reduce_scatter(l, stream=comp)

    hist = 16 if args.fp8_scaling == "delayed" else 0

    def step():
        if wl["fp8"]:
            F.precompute_fp8_scales(mesh, layers, stream=comp, history_len=hist)
        (step_train if args.step == "train" else step_unit)()

    # algorithmic bytes per step per rank: all-gather outputs + fp32 RS inputs
    slot_b = [(l.S_bytes_fp8 if wl["fp8"] else 2 * l.S) for l in layers]
    if args.step == "train":
        n_unshard = [2 if (i not in kept) else 1 for i in range(len(blocks))] + [2]
    else:
        n_unshard = [1] * len(layers)
    bytes_rank = sum(k * W * sb + 4 * W * l.S for k, sb, l in zip(n_unshard, slot_b, layers))

    # physical NVLink bytes this rank sends per step, per direction (the metric's
    # fp32 RS bytes are not what the P2P path puts on the wire).  P2P: the push stores this
    # rank's cast rows into W-1 peers; the reduce-scatter moves this rank's bf16 grad rows of
    # every peer's chunk (store) / every peer's rows of this rank's chunk (pull), (W-1) x own
    # rows x 2 B either way.  NCCL ring: (W-1) x slot bytes (AG) + (W-1) x 4S (fp32 RS).
    # HSDP adds the fp32 replica all-reduce (NCCL ring, 2 (R-1)/R x 4S); the HSDP world pull
    # instead reads this rank's bf16 rows from all R W - 1 other ranks, (R W - 1) x own x 2 B.
    R = mesh.replicate_size if N > 1 else 1

    def wire_unit(l, k):
        if W == 1 and R == 1:
            return 0
        own = [m["row_count"] * m["rest"] for m in l.metas]
        if N > 1 and mesh.algo == "p2p":
            es = [1 if (wl["fp8"] and e) else 2 for e in l.fp8_eligible]
            b = k * (W - 1) * sum(o * s for o, s in zip(own, es))
        else:
            sb = l.S_bytes_fp8 if wl["fp8"] else 2 * l.S
            b = k * (W - 1) * sb
        if hsdp_2ph:   # pieces: (RW-1) x own/R bf16 rows in, then (R-1) fp32 pieces of own/R
            b += (R * W - 1) * 2 * sum(own) // R + (R - 1) * 4 * sum(own) // R
        elif hsdp_wp:
            b += (R * W - 1) * 2 * sum(own)
        elif N > 1 and mesh.algo == "p2p":
            b += (W - 1) * 2 * sum(own)
        else:
            b += (W - 1) * 4 * l.S
        if R > 1 and not hsdp_wp:
            b += 2 * (R - 1) * 4 * l.S // R
        return b
    wire_rank = sum(wire_unit(l, k) for k, l in zip(n_unshard, layers))

    def barrier():
        if N > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        step()
    comp.synchronize()
    mesh.synchronize(600000)
    barrier()
    torch.cuda.synchronize()

    mem = {k: round(v / 2 ** 30, 3) for k, v in mesh.memory().items()}   # after warm-up: pools at steady size
    free_b, total_b = torch.cuda.mem_get_info(dev)
    mem["device_used_GiB"] = round((total_b - free_b) / 2 ** 30, 2)
    mem["device_total_GiB"] = round(total_b / 2 ** 30, 2)
    mem["unit"] = "GiB per rank (peer_mapped: address space of W-1 peers' symmetric buffers, not local HBM)"
    timed_step, graph_prof = step, None
    if args.graph:
        # one eager profiled step: the per-step kernel counts / bytes (no timing events exist
        # inside a graph), then capture the step and time graph.replay() instead
        mesh.profile_enable(True)
        mesh.profile_read(reset=True)
        step()
        comp.synchronize()
        graph_prof = mesh.profile_read(reset=True)
        mesh.profile_enable(False)
        barrier()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=comp):
            step()

        def timed_step():
            with torch.cuda.stream(comp):   # replay() launches on the current stream
                g.replay()
        for _ in range(args.warmup):
            timed_step()
        torch.cuda.synchronize()
        barrier()

    clocks = ClockSampler(list(range(N))) if rank == 0 else None
    if clocks:
        clocks.start()
    mesh.profile_enable(True)
    mesh.profile_read(reset=True)
    # before each iteration a host barrier over ranks + device sync, so all
    # ranks start aligned; CUDA events on the launching stream bracket every step; the step
    # time is the max over ranks per step, `ms_per_step` their mean.  queue_ahead(): a ~50 us
    # device sleep on the compute stream before the start event, so the host has enqueued
    # the step's first launches when the clock starts (as in back-to-back training steps)
    # instead of timing a launch from an idle GPU (~40 us: the whole toy step's size)
    def queue_ahead():
        with torch.cuda.stream(comp):
            torch.cuda._sleep(100_000)   # cycles (~50 us at 1.9-2.0 GHz)

    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        barrier()
        torch.cuda.synchronize()
        queue_ahead()
        ev_a[k].record(comp)
        timed_step()
        ev_b[k].record(comp)
    comp.synchronize()
    torch.cuda.synchronize()
    barrier()
    prof = mesh.profile_read(reset=True)
    mesh.profile_enable(False)
    clk = clocks.stop() if clocks else None
    per_step = [ev_a[k].elapsed_time(ev_b[k]) for k in range(args.steps)]
    t = torch.tensor([0.0] + per_step, device=dev, dtype=torch.float64)
    if N > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t[0] = t[1:].mean()
    ms_max = float(t[0].item())
    step_pct = {"median": round(float(t[1:].median().item()), 4),
                "p10": round(float(torch.quantile(t[1:], 0.1).item()), 4),
                "p90": round(float(torch.quantile(t[1:], 0.9).item()), 4), "of": "per-step max over ranks"}
    value = N * bytes_rank / (ms_max * 1e-3) / 1e9
    algbw_rank = bytes_rank / (ms_max * 1e-3) / 1e9
    busbw_rank = algbw_rank * (W - 1) / W
    prof_step = prof
    if graph_prof is not None:   # replays: one eager step's counts x steps, device time unknown per kernel
        prof_step = {k: {"launches": v["launches"] * args.steps, "ms": 0.0, "bytes": v["bytes"] * args.steps}
                     for k, v in graph_prof.items()}

    # ---- roofline pass: the same step with every unit issued serially (no prefetch), so
    # no two of our kernels overlap and each kernel's event-timed duration is its own
    # (in the prefetch step the unshard of unit i+1 and the reduce-scatter of unit i share
    # HBM / NVLink, which inflates both durations while the step as a whole runs faster)
    # The same pass doubles as the ISOLATED step of SURVEY.md 8(d) (each unit's unshard and
    # reduce-scatter issued and waited one after another, no cross-unit overlap), timed per
    # step like the pipelined one, so both numbers come from one run.
    roof_steps = max(3, min(args.steps, 6))
    serial_saved = args.serial
    args.serial = args.step == "unit"
    step()
    comp.synchronize()
    barrier()
    mesh.profile_enable(True)
    mesh.profile_read(reset=True)
    iso = []
    for _ in range(roof_steps):
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        queue_ahead()
        a.record(comp)
        step()
        b.record(comp)
        iso.append((a, b))
    comp.synchronize()
    prof = mesh.profile_read(reset=True)
    mesh.profile_enable(False)
    args.serial = serial_saved
    ti = torch.tensor([a.elapsed_time(b) for a, b in iso], device=dev, dtype=torch.float64)
    if N > 1:
        dist.all_reduce(ti, op=dist.ReduceOp.MAX)
    ms_iso = float(ti.mean().item())
    barrier()
    proxy = None
    if T:   # the same GEMMs alone, each unit's weights unsharded beforehand (outside the events)
        ms_c = 0.0
        for rep in range(2):
            tot = 0.0
            for l in layers:
                F.fsdp_unshard(l, pdtype, stream=comp)
                F.fsdp_wait_unshard(l, stream=comp)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(comp)
                compute(l.unsharded_params())
                b.record(comp)
                F.fsdp_reshard(l, stream=comp)
                b.synchronize()
                tot += a.elapsed_time(b)
            ms_c = tot          # second repetition: warm GEMM heuristics
        tc = torch.tensor([ms_c], device=dev, dtype=torch.float64)
        if N > 1:
            dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        flops = 6 * T * sum(int(np.prod(s)) for l in layers for s in l.shapes if len(s) == 2)
        proxy = {"tokens": T, "flops_per_step": flops, "ms_compute_only": round(float(tc.item()), 4),
                 "ms_with_fsdp": round(ms_max, 4), "exposed_comm_ms": round(ms_max - float(tc.item()), 4),
                 "compute_TFLOPs": round(flops / (float(tc.item()) * 1e-3) / 1e12, 1)}

    # ---- roofline of the dominant kernel (largest total device time among ours).
    # HBM-bound kernels are measured against the measured HBM copy peak; the fused P2P
    # kernels are NVLink-bound: their bytes are the per-rank NVLink bytes, measured against
    # the measured per-direction peer bandwidth (B200_PROFILING.md: 770 GB/s; 900 nominal).
    peak, peak_src = measured_peaks()
    hbm_k = ["copy_in", "copy_out", "rs_copy_in", "rs_copy_out", "amax", "scale", "stage_grads", "rs_reduce"]
    nvl_k = ["unshard_push", "rs_pull", "rs_scatter", "replica_gather"]
    ours = hbm_k + nvl_k + ["handshake"]
    dom = max(hbm_k + nvl_k, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    per_launch_bytes = d["bytes"] / max(d["launches"], 1)
    avg_ms = d["ms"] / max(d["launches"], 1)
    achieved = per_launch_bytes / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else 0.0
    mech = None
    if dom in nvl_k:
        bound, peak, peak_src = "nvlink", 770.0, "measured peer copy per direction (B200_PROFILING.md; 900 nominal)"
        # what SM-issued traffic (stores for the push, loads for the pull) reaches in the same
        # bidirectional / all-to-all pattern on this pool (profiles/nvlink_ceiling.json)
        try:
            ceil = json.load(open(os.path.join(ROOT, "profiles", "nvlink_ceiling.json")))
            tab = ceil["bidir_2gpu"] if W == 2 else ceil["a2a_4gpu"]
            key = "sm_store" if dom in ("unshard_push", "rs_scatter") else "sm_load"
            mech = {"mechanism": key, "GBps": tab[key], "frac": round(achieved / tab[key], 4),
                    "pattern": "bidirectional, 2 GPUs" if W == 2 else "all-to-all, 4 GPUs",
                    "source": "profiles/nvlink_ceiling.json (scripts/nvlink_probe.cu)"}
        except (OSError, KeyError, ValueError):
            mech = None
    else:
        bound = "hbm"
    def ktable(pr, nsteps, step_ms):
        out = {}
        for k in ours + ["all_gather", "reduce_scatter", "all_reduce"]:
            if pr[k]["launches"]:
                out[k] = {"launches": pr[k]["launches"], "avg_us": round(pr[k]["ms"] / pr[k]["launches"] * 1e3, 2),
                          "GBps": round(pr[k]["bytes"] / (pr[k]["ms"] * 1e-3) / 1e9, 1) if pr[k]["ms"] and pr[k]["bytes"] else None,
                          "share_of_step": round(pr[k]["ms"] / nsteps / step_ms, 4) if step_ms else None}
        return out

    kernels = ktable(prof_step, args.steps, ms_max)            # in the timed (prefetch) step
    kernels_serial = ktable(prof, roof_steps, None)           # roofline pass
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(f"{args.workload}/w{N}", {}).get(dom)
        except Exception:
            traffic = None
    traffic_src = "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/ncu_traffic.json)" \
        if traffic is not None else None
    if traffic is None and bound == "nvlink":
        # NVLink wire bytes: ncu nvltx / nvlrx user-payload bytes per launch of the same kernel
        # on the 8B block at this W, as a ratio to its algorithmic bytes (profiles/round2)
        try:
            wire = json.load(open(os.path.join(ROOT, "profiles", "round2", "nvlink_wire.json")))
            kname = {"unshard_push": "k_unshard_push_bulk", "rs_pull": "k_rs_pull_bulk",
                     "rs_scatter": "k_rs_scatter"}[dom]
            ent = wire[f"W{W}"][kname]
            traffic = int(round(per_launch_bytes * ent["ratio"]))
            traffic_src = (f"NVLink wire bytes: ncu {'nvlrx' if dom == 'rs_pull' else 'nvltx'}__bytes_data_user.sum / "
                           f"algorithmic = {ent['ratio']} for {kname} at W={W} (profiles/round2/nvlink_wire.json) "
                           "x this line's algorithmic bytes per launch")
        except (OSError, KeyError, ValueError):
            traffic = None
    gpu_launches = sum(prof_step[k]["launches"] for k in ours)
    # whole-step HBM efficiency of our kernels in the timed step (sum of their algorithmic
    # HBM bytes / step time), meaningful where no NVLink kernel runs (W = 1)
    step_hbm = sum(prof_step[k]["bytes"] for k in hbm_k) / args.steps / (ms_max * 1e-3) / 1e9

    # ---- e2e through the public API with host buffers (pinned), copies inside the timing
    e2e = None
    if not args.no_e2e:
        bytes_unit = sum(W * sb + 4 * W * l.S for sb, l in zip(slot_b, layers))   # e2e runs the unit step
        e2e = run_e2e(args, F, torch, dist, mesh, layers, grads, comp, dev, N, W, pdtype, wl, bytes_unit,
                      barrier)

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(args, W, full_block=(N == 1))
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max, 4), "ms_per_step_pct": step_pct,
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp8_e4m3+bf16/f32" if wl["fp8"] else "bf16/f32",
            "data": "synthetic (seeded normal params and bf16 grads, Llama 3.1 parameter shapes)",
            "config": {"workload": f"{args.workload} layout: {len(layers)} FSDP units "
                                   f"({'32 blocks + root' if args.workload.startswith('llama3.1-8b') else 'see DESIGN.md'}), "
                                   f"{('fp8 e4m3 (' + args.fp8_scaling + ' scaling)') if wl['fp8'] else 'bf16'} "
                                   f"all-gather / fp32 reduce-scatter, "
                                   f"{'serial' if args.serial else 'prefetch next unit'}",
                       "world_size": N, "shard_size": W, "units": len(layers), "collectives": algo,
                       "step": args.step + (" zero2" if args.zero2 else ""),
                       "cuda_graph": bool(args.graph),
                       "grads": "layer symmetric grad buffers (zero-copy RS)" if lib_grads else "torch tensors (RS stages them)",
                       "l2": "inputs larger than L2 (every unit's shard/grads/buffers are 100s of MB; 126 MB L2)",
                       "bytes_per_step_per_rank": bytes_rank},
            "per_rank": {"algbw_GBps": round(algbw_rank, 2), "busbw_GBps": round(busbw_rank, 2),
                         "busbw_frac_nvlink_900": round(busbw_rank / NVLINK_GBS, 4),
                         "busbw_note": "metric units: counts the paper's fp32 reduce-scatter bytes; the P2P "
                                       "path sends bf16 grads (DESIGN.md R14), so see `wire` for the link rate"},
            "wire": wire_report(wire_rank, ms_max, ms_iso, W, R, hsdp_wp),
            "isolated": {"ms_per_step": round(ms_iso, 4), "steps": roof_steps,
                         "value": round(N * bytes_rank / (ms_iso * 1e-3) / 1e9, 2),
                         "what": "same step with every unit's unshard and reduce-scatter issued serially (no "
                                 "prefetch / cross-unit overlap), per-step barrier, max over ranks"
                                 if args.step == "unit" else "train step (already serial per unit)"},
            "kernels": kernels,
            "kernels_serial": kernels_serial,
            "roofline": {"bound": bound, "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
                         "bytes_per_launch": int(per_launch_bytes), "traffic": traffic, "traffic_source": traffic_src,
                         "sm_mechanism_ceiling": mech,
                         "frac_of_nominal": round(achieved / (NVLINK_GBS if bound == "nvlink" else HBM_NOMINAL_GBS), 4),
                         "nominal_peak": NVLINK_GBS if bound == "nvlink" else HBM_NOMINAL_GBS,
                         "pass": f"serial issue, {roof_steps} steps after the timed region (CUDA events on the launching streams)",
                         "step_hbm_GBps": round(step_hbm, 1), "step_hbm_frac": round(step_hbm / measured_peaks()[0], 4),
                         "step_hbm_frac_of_nominal": round(step_hbm / HBM_NOMINAL_GBS, 4)},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": gpu_launches, "clocks": clk, "memory": mem,
        }
        if proxy:
            line["compute_proxy"] = proxy
            line["config"]["step"] += f" + compute proxy ({T} tokens/rank; value includes compute time)"
    for l in layers:
        l.destroy()
    mesh.destroy()
    if N > 1:
        dist.destroy_process_group()
    return line


def run_e2e(args, F, torch, dist, mesh, layers, grads, comp, dev, N, W, pdtype, wl, bytes_rank, barrier):
    """Same step through the public API, inputs (this step's full grads) copied H2D from
    pinned host memory and the result (every unit's sharded fp32 grad) read back D2H,
    all inside the timed region."""
    max_g = max(sum(g.numel() for g in gs) for gs in grads)
    max_s = max(l.S for l in layers)
    h_in = torch.empty(max_g, dtype=torch.bfloat16).pin_memory()
    big = max(range(len(grads)), key=lambda i: sum(g.numel() for g in grads[i]))
    h_in.copy_(torch.cat([g.view(-1) for g in grads[big]]).cpu())
    h_out = torch.empty(max_s, dtype=torch.float32).pin_memory()
    h2d = sum(sum(g.numel() for g in gs) * 2 for gs in grads)
    d2h = sum(4 * l.S for l in layers)

    h2d_s = torch.cuda.Stream(device=dev)   # PCIe host->device (copy engine)
    d2h_s = torch.cuda.Stream(device=dev)   # PCIe device->host, other direction, overlaps
    n = len(layers)

    def step():
        start = torch.cuda.Event()
        start.record(comp)
        h2d_s.wait_event(start)
        ev_in = []
        with torch.cuda.stream(h2d_s):
            for i in range(n):           # this step's input: every unit's full grads, H2D
                off = 0
                for g in grads[i]:
                    g.view(-1).copy_(h_in[off:off + g.numel()], non_blocking=True)
                    off += g.numel()
                e = torch.cuda.Event()
                e.record(h2d_s)
                ev_in.append(e)
        if wl["fp8"]:
            F.precompute_fp8_scales(mesh, layers, stream=comp, history_len=16 if args.fp8_scaling == "delayed" else 0)
        with torch.cuda.stream(comp):
            F.fsdp_unshard(layers[0], pdtype, stream=comp)
            for i in range(n):
                F.fsdp_wait_unshard(layers[i], stream=comp)
                if i + 1 < n:
                    F.fsdp_unshard(layers[i + 1], pdtype, stream=comp)
                F.fsdp_reshard(layers[i], stream=comp)
                comp.wait_event(ev_in[i])
                F.reduce_scatter_grads(layers[i], grads[i], stream=comp)
                # the step's result: the unit's sharded fp32 grad, D2H as soon as it is reduced
                F.fsdp_wait_reduce_scatter(layers[i], stream=d2h_s)
                with torch.cuda.stream(d2h_s):
                    h_out[:layers[i].S].copy_(layers[i].sharded_grad_flat(), non_blocking=True)
        done = torch.cuda.Event()
        done.record(d2h_s)
        comp.wait_event(done)
        comp.wait_stream(h2d_s)

    step()
    comp.synchronize()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(comp)
    for _ in range(args.e2e_steps):
        step()
    e1.record(comp)
    comp.synchronize()
    ms = e0.elapsed_time(e1) / args.e2e_steps
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    if N > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": round(N * bytes_rank / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "steps": args.e2e_steps, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


# ----------------------------------------------------------------------------- oracle (CPU)
def _oracle_sample(model: str, W: int, full_block: bool = False):
    """Bounded sample of the workload for the CPU oracle: one Llama block (full_block; 218.1M
    params for 8B, ~15 s of single-threaded NumPy on the GPU host) or its attention weights +
    norms (41.9M params, ~3 s), all W ranks simulated."""
    import synth
    u = synth.model_units(model, include_root=False)[0]
    keep = [i for i, (n, _, _) in enumerate(u) if full_block or n.startswith("attention")]
    shapes = [u[i][1] for i in keep]
    elig = [u[i][2] for i in keep]
    params = [synth.param_values(0, p, s) for p, s in enumerate(shapes)]
    grads = [[synth.grad_bf16_bits(0, p, q, s) for p, s in enumerate(shapes)] for q in range(W)]
    return shapes, elig, params, grads


def _oracle_step(World, BF16, FP8, shapes, elig, params, grads, W, fp8):
    w = World(shapes, W, elig)
    shards = w.shard(params)
    if fp8:
        _, scale = w.precompute_fp8_scales(shards)
        w.unshard(shards, FP8, scale)
    else:
        w.unshard(shards, BF16)
    w.reduce_scatter_grads(grads, BF16, True)
    slot = w.S_bytes_fp8 if fp8 else 2 * w.S
    return W * (W * slot + 4 * W * w.S)     # same algorithmic bytes, all simulated ranks


def host_info():
    """CPU model, RAM, core counts of the host the CPU baseline ran on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        import psutil
        ram = round(psutil.virtual_memory().total / 2 ** 30, 1)
    except Exception:   # noqa: BLE001
        pass
    return {"cpu_model": model, "ram_GiB": ram, "os_cpu_count": os.cpu_count(),
            "affinity_cores": len(os.sched_getaffinity(0))}


def cpu_baseline(args, W, full_block=True):
    """The unchanged oracle on a bounded sample of the workload, rank 0's host cores.  N = 1:
    one full block (~15 s) plus the all-cores run; N > 1: the block's attention weights +
    norms with all W ranks simulated (the oracle's work grows with W; bounded to ~10-30 s)."""
    from oracle import World
    from oracle.world import BF16, FP8
    wl = WORKLOADS[args.workload]
    shapes, elig, params, grads = _oracle_sample(wl["model"], W, full_block=full_block)
    t0 = time.perf_counter()
    nbytes = _oracle_step(World, BF16, FP8, shapes, elig, params, grads, W, wl["fp8"])
    dt = time.perf_counter() - t0
    what = "block" if full_block else "block's attention weights + norms"
    out = {"value": round(nbytes / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
           "seconds": round(dt, 2),
           "sample": f"one {wl['model']} {what} ({sum(int(np.prod(s)) for s in shapes)} params), "
                     f"W={W} simulated ranks, {'fp8' if wl['fp8'] else 'bf16'} unshard + fp32 reduce-scatter, "
                     f"single-threaded NumPy",
           "host": host_info()}
    if full_block:
        out["all_cores"] = _cpu_all_cores(wl, W)
    return out


def _oracle_worker(model, W, fp8):
    """One process of the all-cores CPU baseline: the unchanged oracle on a bounded sample."""
    from oracle import World
    from oracle.world import BF16, FP8
    shapes, elig, params, grads = _oracle_sample(model, W, full_block=False)
    return _oracle_step(World, BF16, FP8, shapes, elig, params, grads, W, fp8)


def _cpu_all_cores(wl, W, max_procs=16):
    """SURVEY.md 8(d) "two runs: single-threaded and all cores": the unchanged oracle run
    as k independent processes at once (one bounded sample each, like independent units),
    k = min(usable cores, 16); GB/s = the bytes of all k samples / wall time."""
    import concurrent.futures as cf
    import multiprocessing as mp
    try:
        k = max(1, min(len(os.sched_getaffinity(0)), max_procs))
        ctx = mp.get_context("spawn")
        t0 = time.perf_counter()
        with cf.ProcessPoolExecutor(max_workers=k, mp_context=ctx) as ex:
            total = sum(ex.map(_oracle_worker, [wl["model"]] * k, [W] * k, [wl["fp8"]] * k))
        dt = time.perf_counter() - t0
        return {"value": round(total / dt / 1e9, 4), "unit": "GB/s", "cores": k, "kind": "oracle",
                "seconds": round(dt, 2),
                "sample": f"{k} processes x one {wl['model']} block's attention weights + norms, W={W} "
                          f"simulated ranks each (wall time incl. process start)"}
    except Exception as e:   # noqa: BLE001 (a reported baseline only)
        return {"error": f"{type(e).__name__}: {str(e)[:120]}"}


def run_reference(args):
    N = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import World
    from oracle.world import BF16, FP8
    wl = WORKLOADS[args.workload]
    W = args.gpus
    shapes, elig, params, grads = _oracle_sample(wl["model"], W)
    for _ in range(args.warmup):
        _oracle_step(World, BF16, FP8, shapes, elig, params, grads, W, wl["fp8"])
    t0 = time.perf_counter()
    nbytes = 0
    for _ in range(args.steps):
        nbytes += _oracle_step(World, BF16, FP8, shapes, elig, params, grads, W, wl["fp8"])
    dt = time.perf_counter() - t0
    value = nbytes / dt / 1e9
    sample = (f"one {wl['model']} block's attention weights + norms per step, W={W} simulated ranks, "
              f"unshard + reduce-scatter, single-threaded NumPy oracle")
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32 (numpy)",
            "data": "synthetic", "config": {"workload": f"{args.workload} (bounded oracle sample)", "world_size": W},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launcher_cmd(argv, n: int, port: int):
    """The torchrun command a plain `python bench.py --gpus N` (N > 1, no WORLD_SIZE in the
    environment) re-executes itself under: one rank per GPU on this node, rendezvous on
    127.0.0.1, the same arguments."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: launch our own N ranks; rank 0 prints the JSON line
        res = subprocess.run(launcher_cmd(sys.argv[1:], args.gpus, _free_port()), cwd=ROOT)
        raise SystemExit(res.returncode)
    line = run_reference(args) if args.impl == "reference" else run_ours(args)
    if line is not None:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")


if __name__ == "__main__":
    main()
