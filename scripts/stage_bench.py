#!/usr/bin/env python3
"""Per-stage kernel timings on ONE GPU at the Llama 3.1 8B (or 70B) block layout for
W = 1, 2, 4, 8 ("W=1: K1-K6 GB/s and fraction of HBM; also the
K2/K4/K5 layouts for W = 2, 4, 8 on one GPU"), each next to the torch op FSDP2 uses for the
same step (timed on the same box as context, 8(d) "Timing protocol"):

    K1  local amax          vs torch._foreach_norm(shards, inf) + stack
    K2  copy-in bf16        vs torch._foreach_copy_ (fp32 -> bf16 views of the AG slot)
    K3  copy-in fp8         (no single torch op: per-param mul + clamp + .to(e4m3) + foreach copy)
    K4  copy-out bf16       vs torch.split_with_sizes_copy(ag.view(W, S), n_p, dim=1, out=...)
    K5  RS copy-in          vs torch._chunk_cat(grads, 0, W, out=rs_in.view(W, S)) + rs_in.div_(W)
    K6  RS copy-out (copy)  vs Tensor.copy_
    push (P2P unshard, W arenas on this GPU) and pull (P2P reduce, W stagings on this GPU):
        the fused kernels with every peer pointer local, i.e. their HBM-only cost.

Every rank's stage runs on a communicator-less local mesh (rank 0's slot).  Each timed
iteration is preceded by an L2 flush (a 512 MB write) outside the event pair; per-iteration
CUDA-event times -> median / p10 / p90.  GB/s = algorithmic bytes (DESIGN.md kernel table)
/ median time; frac = GB/s / MEASURED_PEAKS.json HBM.  One JSON line per (W, stage, impl).

    python scripts/stage_bench.py [--model llama3.1-8b] [--ws 1,2,4,8] [--iters 20] [--out f]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2410_06511_b200 as F  # noqa: E402


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k in ("hbm_gbs", "hbm_gbps", "hbm_GBps"):
            if k in d:
                return float(d[k]), "MEASURED_PEAKS.json"
        for k, v in d.items():
            if "hbm" in k.lower() and isinstance(v, (int, float)):
                return float(v), "MEASURED_PEAKS.json:" + k
    except (OSError, ValueError):
        pass
    return 6542.7, "DESIGN.md measured copy bandwidth"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3.1-8b", choices=["llama3.1-8b", "llama3.1-70b", "toy"])
    ap.add_argument("--ws", default="1,2,4,8")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--no-torch", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    peak, peak_src = hbm_peak()
    st = torch.cuda.Stream(device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    lines = []

    def timed(fn):
        with torch.cuda.stream(st):
            for _ in range(args.warmup):
                fn()
            ts = []
            for _ in range(args.iters):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
        ts = np.array(ts)
        return float(np.median(ts)), float(np.percentile(ts, 10)), float(np.percentile(ts, 90))

    def emit(W, stage, impl, nbytes, fn, note=None):
        try:
            med, p10, p90 = timed(fn)
        except (RuntimeError, TypeError) as e:      # a torch op that does not exist / accept this
            lines.append({"W": W, "stage": stage, "impl": impl, "error": str(e).splitlines()[0][:160]})
            print(json.dumps(lines[-1]), flush=True)
            return
        gbps = nbytes / (med * 1e-3) / 1e9
        d = {"model": args.model, "W": W, "stage": stage, "impl": impl, "bytes": int(nbytes),
             "ms_median": round(med, 5), "ms_p10": round(p10, 5), "ms_p90": round(p90, 5),
             "GBps": round(gbps, 1), "frac_hbm": round(gbps / peak, 4)}
        if note:
            d["note"] = note
        lines.append(d)
        print(json.dumps(d), flush=True)

    unit = synth.model_units(args.model)[0]
    shapes = [tuple(s) for _, s, _ in unit]
    elig = [bool(e) for _, _, e in unit]
    numels = [int(np.prod(s)) for s in shapes]
    N = sum(numels)
    g = torch.Generator(device=dev)
    g.manual_seed(241006511)
    for W in [int(x) for x in args.ws.split(",")]:
        mesh = F.Mesh(W, 0, 0, local=True)
        layer = F.fsdp_shard(mesh, None, elig, shapes=shapes)
        S, M = layer.S, layer.metas
        layer.sharded_flat().normal_(0, 0.02, generator=g)
        n_p = [m["padded_numel"] for m in M]
        off = [m["elem_offset"] for m in M]
        valid = [m["row_count"] * m["rest"] for m in M]
        n_fp8 = sum(n for n, e in zip(n_p, elig) if e)
        packed = sum(n_p) == S          # FSDP2's packing (no alignment gaps) == ours
        shard_v = [layer.sharded_param(p, padded=True).view(-1) for p in range(layer.P)]

        # K1 + K1b: local amax over fp8-eligible shards, then the scales
        amax = torch.zeros(layer.P, dtype=torch.float32, device=dev)
        scale = torch.zeros_like(amax)
        emit(W, "K1_amax", "ours", 4 * n_fp8, lambda: F.stage_local_amax(layer, amax, stream=st))
        F.stage_local_amax(layer, amax, stream=st)
        emit(W, "K1b_scale", "ours", 8 * layer.P, lambda: F.stage_fp8_scale(layer, amax, scale, stream=st))
        if not args.no_torch:
            ev = [v for v, e in zip(shard_v, elig) if e]
            emit(W, "K1_amax", "torch._foreach_norm(inf)", 4 * n_fp8,
                 lambda: torch.stack(torch._foreach_norm(ev, float("inf"))))
        st.synchronize()

        # K2 copy-in bf16 into rank 0's slot of a [W][S] AG buffer
        ag = torch.empty(W * S, dtype=torch.bfloat16, device=dev)
        emit(W, "K2_copy_in_bf16", "ours", 6 * S, lambda: F.stage_copy_in(layer, torch.bfloat16, ag[:S], stream=st))
        if not args.no_torch:
            dsts = [ag[o:o + n] for o, n in zip(off, n_p)]
            emit(W, "K2_copy_in_bf16", "torch._foreach_copy_", 6 * S, lambda: torch._foreach_copy_(dsts, shard_v))
        # K3 copy-in fp8 (mixed: e4m3 linears, bf16 norms)
        slot8 = torch.empty(layer.S_bytes_fp8, dtype=torch.uint8, device=dev)
        emit(W, "K3_copy_in_fp8", "ours", 4 * S + layer.S_bytes_fp8,
             lambda: F.stage_copy_in(layer, torch.float8_e4m3fn, slot8, fp8_scales=scale, stream=st))
        if not args.no_torch:
            def torch_fp8():
                for p in range(layer.P):
                    if elig[p]:
                        shard_v[p].mul(scale[p]).clamp_(-448, 448).to(torch.float8_e4m3fn)
                    else:
                        shard_v[p].to(torch.bfloat16)
            emit(W, "K3_copy_in_fp8", "torch mul+clamp+to (per param)", 4 * S + layer.S_bytes_fp8, torch_fp8,
                 note="cast only, no copy into the slot: a lower bound for the eager path")

        # K4 copy-out bf16 from the full [W][S] buffer into per-param full tensors
        ag.normal_(generator=g)
        outs = [torch.empty(s, dtype=torch.bfloat16, device=dev) for s in shapes]
        emit(W, "K4_copy_out_bf16", "ours", 4 * N, lambda: F.stage_copy_out(layer, torch.bfloat16, ag, outs, stream=st))
        if not args.no_torch and packed and all(v == n for v, n in zip(numels, [W * x for x in n_p])):
            ov = [o.view(W, -1) for o in outs]
            emit(W, "K4_copy_out_bf16", "torch.split_with_sizes_copy", 4 * N,
                 lambda: torch.split_with_sizes_copy(ag.view(W, S), n_p, dim=1, out=ov))
        del outs

        # K5 RS copy-in: bf16 full grads -> fp32 [W][S] / W
        grads = [torch.empty(s, dtype=torch.bfloat16, device=dev).normal_(0, 1e-3, generator=g) for s in shapes]
        rs_in = torch.empty(W * S, dtype=torch.float32, device=dev)
        emit(W, "K5_rs_copy_in", "ours", 2 * N + 4 * W * S,
             lambda: F.stage_rs_copy_in(layer, grads, torch.float32, True, rs_in, stream=st))
        if not args.no_torch and packed:
            rv = rs_in.view(W, S)

            def chunk_cat():
                torch._chunk_cat(grads, dim=0, num_chunks=W, out=rv)
                rs_in.div_(W)
            emit(W, "K5_rs_copy_in", "torch._chunk_cat+div_", 2 * N + 4 * W * S, chunk_cat,
                 note="FSDP2 chunk_cat (casting into the fp32 out) then one division kernel (P:466)")
        # K6 RS copy-out (copy mode, fp32)
        emit(W, "K6_rs_copy_out", "ours", 8 * S,
             lambda: F.stage_rs_copy_out(layer, rs_in[:S], torch.float32, False, stream=st))
        if not args.no_torch:
            dst = layer.sharded_grad_flat()
            emit(W, "K6_rs_copy_out", "torch copy_", 8 * S, lambda: dst.copy_(rs_in[:S]))
        del rs_in
        torch.cuda.empty_cache()

        # fused P2P kernels with every peer arena on this GPU (HBM-only cost)
        _, arena_bytes = F.unsharded_layout(layer, torch.bfloat16)
        arenas = [torch.empty(arena_bytes, dtype=torch.uint8, device=dev) for _ in range(W)]
        emit(W, "push_bf16", "ours", 4 * S + 2 * W * sum(valid),
             lambda: F.stage_unshard_push(layer, torch.bfloat16, arenas, stream=st),
             note="cast the shard once, store it into all W arenas (all local here)")
        del arenas
        soffs, stot = F.grad_staging_layout(layer)
        staging = torch.empty(stot, dtype=torch.bfloat16, device=dev)
        F.stage_grads_to_staging(layer, grads, staging, stream=st)
        emit(W, "grads_to_staging", "ours", 4 * N,
             lambda: F.stage_grads_to_staging(layer, grads, staging, stream=st))
        # W distinct stagings (the same buffer W times would serve W-1 of the reads from L2)
        stagings = [staging] + [staging.clone() for _ in range(W - 1)]
        emit(W, "pull_fp32", "ours", 2 * W * sum(valid) + 4 * S,
             lambda: F.stage_rs_pull(layer, stagings, torch.bfloat16, stream=st),
             note="reads this rank's rows from W distinct stagings (all local here), fp32 sum, /W")
        del staging, stagings
        # store-based reduce-scatter: scatter into W receive buffers (all local here), then
        # the local ascending-rank reduce of this rank's receive buffer
        recvs = [torch.empty(W * S, dtype=torch.bfloat16, device=dev) for _ in range(W)]
        emit(W, "rs_scatter", "ours", 4 * N, lambda: F.stage_rs_scatter(layer, grads, recvs, stream=st),
             note="this rank's rows of every rank's chunk -> W receive buffers (all local here)")
        F.stage_rs_scatter(layer, grads, recvs, stream=st)
        emit(W, "rs_recv_reduce", "ours", sum(valid) * (2 * W + 4),
             lambda: F.stage_rs_recv_reduce(layer, recvs[0], torch.bfloat16, stream=st),
             note="W slots of bf16 rows -> fp32 grad, /W, ascending-rank sum")
        del recvs, grads
        st.synchronize()
        layer.destroy()
        mesh.destroy()
        torch.cuda.empty_cache()

    meta = {"peak_hbm_GBps": peak, "peak_source": peak_src, "device": torch.cuda.get_device_name(0),
            "l2_flush": "512 MB write before each timed iteration", "iters": args.iters}
    print(json.dumps({"meta": meta}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for d in lines + [{"meta": meta}]:
                f.write(json.dumps(d) + "\n")


if __name__ == "__main__":
    main()
