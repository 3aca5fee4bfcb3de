#!/usr/bin/env python3
"""Copy-engine NVLink schedules (one process, W GPUs): how close cudaMemcpyPeerAsync gets to
the link when every GPU sends to every peer (the unshard / reduce-scatter pattern), under
different issue schedules.  Per GPU per direction GB/s, best of 5, CUDA events.

  concurrent  W-1 streams per GPU, one copy per peer at once (profiles/nvlink_ceiling.json
              a2a_4gpu copy_engine: 397 GB/s at W=4)
  perm        one stream per GPU, peers in the order rank+1, rank+2, ... (at every moment each
              GPU sends to one peer and receives from one: a permutation)
  perm_chunk  one stream, the per-peer data cut into C-byte chunks issued round robin over the
              peers (rank+1 first)
Run: python scripts/ce_probe.py --W 4 [--mib 1024]"""
from __future__ import annotations

import argparse
import json

import torch


def enable_peers(W):
    from cuda.bindings import runtime as rt
    for a in range(W):
        rt.cudaSetDevice(a)
        for b in range(W):
            if a != b:
                rt.cudaDeviceEnablePeerAccess(b, 0)


def copy(dst_t, dst_dev, src_t, src_dev, nbytes, stream):
    """cudaMemcpyPeerAsync on `stream` (raw: torch's cross-device copy_ adds stream syncs on
    the destination device that would serialize the schedules)."""
    from cuda.bindings import runtime as rt
    err = rt.cudaMemcpyPeerAsync(dst_t, dst_dev, src_t, src_dev, nbytes, stream.cuda_stream)[0]
    if int(err) != 0:
        raise RuntimeError(f"cudaMemcpyPeerAsync: {err}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--W", type=int, default=2)
    ap.add_argument("--mib", type=int, default=1024, help="bytes each GPU sends in total")
    ap.add_argument("--chunks", default="4,16,64", help="perm_chunk sizes in MiB")
    args = ap.parse_args()
    W = args.W
    enable_peers(W)
    per_peer = (args.mib << 20) // (W - 1)
    per_peer -= per_peer % 4096
    src = [torch.empty(per_peer * (W - 1), dtype=torch.uint8, device=f"cuda:{r}") for r in range(W)]
    # dst[r][q]: rank r's receive area for rank q's data
    dst = [[torch.empty(per_peer, dtype=torch.uint8, device=f"cuda:{r}") for q in range(W)] for r in range(W)]
    streams = [[torch.cuda.Stream(device=r) for _ in range(W)] for r in range(W)]

    def run(schedule, chunk=0):
        ts = []
        for it in range(6):
            ev = []
            for r in range(W):
                torch.cuda.synchronize(r)
            for r in range(W):
                with torch.cuda.device(r):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    s0 = streams[r][0]
                    a.record(s0)
                    for i in range(1, W):
                        streams[r][i].wait_stream(s0)
                    peers = [(r + k) % W for k in range(1, W)]
                    if schedule == "concurrent":
                        for i, q in enumerate(peers):
                            copy(dst[q][r].data_ptr(), q, src[r].data_ptr() + i * per_peer, r, per_peer,
                                 streams[r][i + 1])
                        for i in range(1, W):
                            s0.wait_stream(streams[r][i])
                    elif schedule == "perm":
                        for i, q in enumerate(peers):
                            copy(dst[q][r].data_ptr(), q, src[r].data_ptr() + i * per_peer, r, per_peer, s0)
                    else:
                        for off in range(0, per_peer, chunk):
                            n = min(chunk, per_peer - off)
                            for i, q in enumerate(peers):
                                copy(dst[q][r].data_ptr() + off, q, src[r].data_ptr() + i * per_peer + off, r, n, s0)
                    b.record(s0)
                    ev.append((a, b))
            for r in range(W):
                torch.cuda.synchronize(r)
            if it:
                ts.append(max(a.elapsed_time(b) for a, b in ev))
        t = min(ts)
        gbs = per_peer * (W - 1) / (t * 1e-3) / 1e9
        rec = {"W": W, "schedule": schedule, "chunk_MiB": chunk >> 20, "ms": round(t, 3),
               "GBps_per_gpu_per_direction": round(gbs, 1), "bytes_per_gpu": per_peer * (W - 1)}
        print(json.dumps(rec), flush=True)

    run("concurrent")
    run("perm")
    for c in args.chunks.split(","):
        run("perm_chunk", int(c) << 20)


if __name__ == "__main__":
    main()
