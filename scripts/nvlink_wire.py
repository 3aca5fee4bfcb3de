#!/usr/bin/env python3
"""NVLink wire bytes and per-direction bandwidth of the fused P2P kernels (VERDICT r1
"next" 3: prove wire bytes ~ algorithmic bytes for push, pull and store-scatter).

ONE process drives W GPUs (W <= visible GPUs): rank r's layer (a communicator-less mesh)
lives on GPU r, every rank's arenas / receive buffers / grad stagings on its own GPU, and
peer access is enabled between all of them, so each stage kernel does exactly what it does
in the multi-process path (16-byte / TMA stores and loads into peers' memory over NVLink)
minus the flag handshakes.  Being one process, the kernels can be profiled with ncu
(kernel replay) without a multi-rank command:

  ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,\
nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:"k_unshard_push|k_rs_pull|k_rs_scatter" --csv python scripts/nvlink_wire.py --W 2 --iters 1

Without ncu it times every kernel with all W ranks launched concurrently (CUDA events per
GPU) and prints one JSON line per kernel: algorithmic NVLink bytes per rank per launch
((W-1) * 2c, c = the rank's own elements) and GB/s per direction.
Workload: one Llama 3.1 8B TransformerBlock (bench.py's unit), bf16 all-gather, bf16 grads
(fp32 reduction)."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_2410_06511_b200 as F  # noqa: E402


def enable_peers(W):
    from cuda.bindings import runtime as rt
    for a in range(W):
        rt.cudaSetDevice(a)
        for b in range(W):
            if a != b:
                err = rt.cudaDeviceEnablePeerAccess(b, 0)[0]
                if int(err) not in (0, 704):   # 704 = already enabled
                    raise RuntimeError(f"peer access {a}->{b}: {err}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, default=2)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--model", default="llama3.1-8b")
    ap.add_argument("--kernels", default="push,scatter,pull,ce")
    args = ap.parse_args()
    W = args.W
    assert torch.cuda.device_count() >= W, f"needs {W} GPUs"
    enable_peers(W)
    u = synth.model_units(args.model, include_root=False)[0]
    shapes = [s for _, s, _ in u]
    elig = [e for _, _, e in u]
    meshes = [F.Mesh(W, r, r, local=True) for r in range(W)]
    layers = []
    for r in range(W):
        torch.cuda.set_device(r)
        layers.append(F.fsdp_shard(meshes[r], None, elig, shapes=shapes))
        layers[-1].sharded_flat().normal_(0.0, 0.02)
    own = [sum(m["row_count"] * m["rest"] for m in l.metas) for l in layers]
    streams = [torch.cuda.Stream(device=r) for r in range(W)]
    kinds = args.kernels.split(",")
    out = []

    def timed(name, launch, nvl_bytes):
        """launch(r, stream) for every rank at once; max over ranks of the event time."""
        for _ in range(2):   # warm-up
            for r in range(W):
                with torch.cuda.device(r):
                    launch(r, streams[r])
            for r in range(W):
                torch.cuda.synchronize(r)
        ts = []
        for _ in range(args.iters):
            ev = []
            for r in range(W):
                with torch.cuda.device(r):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(streams[r])
                    launch(r, streams[r])
                    b.record(streams[r])
                    ev.append((a, b))
            for r in range(W):
                torch.cuda.synchronize(r)
            ts.append(max(a.elapsed_time(b) for a, b in ev))
        t = sorted(ts)[len(ts) // 2]
        rec = {"kernel": name, "W": W, "model": args.model, "ms_median": round(t, 4),
               "nvlink_bytes_per_rank": [int(b) for b in nvl_bytes],
               "GBps_per_direction": round(max(nvl_bytes) / (t * 1e-3) / 1e9, 1),
               "of_770": round(max(nvl_bytes) / (t * 1e-3) / 1e9 / 770.0, 4),
               "of_900": round(max(nvl_bytes) / (t * 1e-3) / 1e9 / 900.0, 4),
               "timing": "all ranks launched at once, one process, max over GPUs of CUDA-event time"}
        out.append(rec)
        print(json.dumps(rec), flush=True)

    if "push" in kinds:
        offs, total = F.unsharded_layout(layers[0], torch.bfloat16)
        arenas = [torch.empty(total, dtype=torch.uint8, device=f"cuda:{d}") for d in range(W)]
        timed("k_unshard_push_bulk",
              lambda r, s: F.stage_unshard_push(layers[r], torch.bfloat16, arenas, stream=s),
              [(W - 1) * 2 * c for c in own])
        del arenas
    if "ce" in kinds:
        # copy-engine variant of the push's transfer (rows already cast): per peer and param one
        # cudaMemcpyPeerAsync of this rank's rows into the peer's arena, on `nce` streams per rank
        from cuda.bindings import runtime as rt
        offs, total = F.unsharded_layout(layers[0], torch.bfloat16)
        arenas = [torch.empty(total, dtype=torch.uint8, device=f"cuda:{d}") for d in range(W)]
        for nce in (1, 2, 4):
            ce_st = [[torch.cuda.Stream(device=r) for _ in range(nce)] for r in range(W)]

            def ce_push(r, s, nce=nce, ce_st=ce_st):
                jobs = []
                for k in range(1, W):
                    q = (r + k) % W
                    for p, m in enumerate(layers[r].metas):
                        n = m["row_count"] * m["rest"] * 2
                        if n:
                            off = offs[p] + m["row_begin"] * m["rest"] * 2
                            jobs.append((arenas[q].data_ptr() + off, q, arenas[r].data_ptr() + off, r, n))
                for st in ce_st[r]:
                    st.wait_stream(s)
                for i, (d, dq, src, sr, n) in enumerate(jobs):
                    err = rt.cudaMemcpyPeerAsync(d, dq, src, sr, n, ce_st[r][i % nce].cuda_stream)[0]
                    assert int(err) == 0, err
                for st in ce_st[r]:
                    s.wait_stream(st)
            timed(f"ce_push_{nce}streams", ce_push, [(W - 1) * 2 * c for c in own])
        del arenas
    grads = []
    for q in range(W):
        g = torch.Generator(device=f"cuda:{q}").manual_seed(q)
        grads.append([(torch.randn(s, generator=g, device=f"cuda:{q}") * 1e-3).to(torch.bfloat16) for s in shapes])
    S = layers[0].S
    if "scatter" in kinds:
        recv = [torch.empty(W * S * 2, dtype=torch.uint8, device=f"cuda:{d}") for d in range(W)]
        # bytes this rank stores into OTHER ranks: its rows of every other rank's chunk
        sc = [sum(sum(layers[d].metas[p]["row_count"] * layers[d].metas[p]["rest"] for p in range(len(shapes)))
                  for d in range(W) if d != q) * 2 for q in range(W)]
        timed("k_rs_scatter", lambda r, s: F.stage_rs_scatter(layers[r], grads[r], recv, stream=s), sc)
        del recv
    if "pull" in kinds:
        offs, total = F.grad_staging_layout(layers[0])
        stag = [torch.empty(total + 64, dtype=torch.bfloat16, device=f"cuda:{q}") for q in range(W)]
        for q in range(W):
            F.stage_grads_to_staging(layers[q], grads[q], stag[q])
        for q in range(W):
            torch.cuda.synchronize(q)
        timed("k_rs_pull", lambda r, s: F.stage_rs_pull(layers[r], stag, torch.bfloat16, torch.float32, True, False,
                                                         stream=s),
              [(W - 1) * 2 * c for c in own])
    for l in layers:
        l.destroy()
    for m in meshes:
        m.destroy()


if __name__ == "__main__":
    main()
