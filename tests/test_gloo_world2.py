"""N>1 host logic on CPU: two processes over torch.distributed gloo (world_size 2).

Each rank computes its Shard(0) layout through the C ABI (host-only), the ranks exchange
layout hashes (the agreement check fsdp_shard performs), rank 0's NCCL unique id is
broadcast (Mesh.from_process_group's bootstrap), and each rank's local view is checked
against the oracle's simulated World(2): rank r's rows equal the oracle's rank-r shard,
and the gathered shards reproduce the full parameters.  The host-collective mesh's
all-gather callback (fsdp_mesh_init_hostcoll) is called as the library calls it."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        import paper_2410_06511_b200 as f
        from oracle import World
        unit = synth.ragged_unit(3, world_size=world) + synth.model_units("toy", include_root=False)[0]
        shapes = [s for _, s, _ in unit]
        elig = [e for _, _, e in unit]
        metas, S, Sb, h = f.layout_compute(shapes, world, rank, elig)
        hs = [None] * world
        dist.all_gather_object(hs, h)
        assert len(set(hs)) == 1, hs
        # a rank with a different unit must be detected by the hash
        bad = f.layout_compute(shapes[:-1] + [(shapes[-1][0] + 1,) + tuple(shapes[-1][1:])], world, rank, elig)[3]
        assert bad != h
        # NCCL unique id bootstrap over the process group (no GPU needed for the id)
        obj = [f.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert len(set(ids)) == 1 and len(ids[0]) == 128
        # local shard = rows of the full params per this rank's metadata; compare with oracle
        params = [synth.param_values(0, p, s) for p, s in enumerate(shapes)]
        w = World(shapes, world, elig)
        oracle_shard = w.shard(params)[rank]
        mine = np.zeros(S, np.float32)
        for m, full in zip(metas, params):
            rows = full.reshape(m["dim0"], m["rest"])[m["row_begin"]:m["row_begin"] + m["row_count"]].reshape(-1)
            mine[m["elem_offset"]:m["elem_offset"] + rows.size] = rows
        np.testing.assert_array_equal(mine, oracle_shard)
        # all-gather of the local shards (gloo) + copy-out by metadata reproduces the params
        t = torch.from_numpy(mine)
        gathered = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        for p, full in enumerate(params):
            pieces = []
            for r in range(world):
                mr = f.layout_compute(shapes, world, r, elig)[0][p]
                pieces.append(gathered[r].numpy()[mr["elem_offset"]:mr["elem_offset"] + mr["row_count"] * mr["rest"]])
            np.testing.assert_array_equal(np.concatenate(pieces).reshape(full.shape), full)
        # the host-collective mesh's all-gather callback (fsdp_host_allgather_fn over gloo),
        # called the way the library calls it: raw host pointers, rank-major output
        import ctypes as C
        from paper_2410_06511_b200.fsdp import _host_allgather
        fn = _host_allgather(dist.group.WORLD)
        for nbytes in (1, 8, 64):   # barrier byte, layout hash, CUDA IPC handle
            send = (C.c_uint8 * nbytes)(*[(rank * 31 + i) & 0xFF for i in range(nbytes)])
            recv = (C.c_uint8 * (nbytes * world))()
            assert fn(C.addressof(send), C.addressof(recv), nbytes, None) == 0
            want = [(r * 31 + i) & 0xFF for r in range(world) for i in range(nbytes)]
            assert list(recv) == want, (nbytes, list(recv)[:16])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_gloo_world2_layout_agreement_and_bootstrap():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
