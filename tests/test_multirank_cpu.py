"""World-size-2 gloo tests of the multi-GPU host logic on CPU:
view shards partition the views, the sum over ranks of the per-shard
backprojections (oracle, allreduced with gloo) equals the full one, every
rank derives the same bit-exact schedule, the NCCL unique id broadcast
path delivers rank 0's bytes, and the peer-handle exchange of NEXT-3 gathers
every rank's blob in rank order."""
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
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ms2g_synth as S
        import oracle as O
        import paper_2203_07308_b200 as P
        n, V, B = 32, 30, 48
        g = O.Geometry(n, V, B)
        vb, ve = P.view_shard(V, rank, world)
        r = S.random_sinogram((V, B), 5).astype(np.float64)
        views = np.arange(vb, ve)
        part = O.backward(g, 2, r[vb:ve], views=views, nthreads=1)
        t = torch.from_numpy(part.copy())
        dist.all_reduce(t)
        full = O.backward(g, 2, r, nthreads=1)
        err = float(np.max(np.abs(t.numpy() - full)) / np.max(np.abs(full)))
        pr = S.PRESETS[3]
        sch = P.schedule(None, pr.stages, pr.option, pr.n_subsets, S.config_seed(3))
        allsch = [None] * world
        dist.all_gather_object(allsch, sch)
        # the NCCL unique id as attach_nccl makes it: rank 0 asks libms2g
        # (ncclGetUniqueId, no GPU needed), the process group broadcasts it
        import ctypes
        L = P.load()
        uid = None
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            assert L.ms2g_nccl_unique_id(buf) == 0
            uid = bytes(buf)
        got = P.broadcast_unique_id(uid, rank, world)
        ids = [None] * world
        dist.all_gather_object(ids, got)
        id_ok = all(i == ids[0] for i in ids) and len(got) == 128 and any(got)
        # the attach entry point validates before touching NCCL or a device
        id_ok &= L.ms2g_attach_nccl(None, (ctypes.c_uint8 * 128).from_buffer_copy(got), rank, world) == 7
        # NEXT-3 peer blob exchange: rank-ordered concatenation of equal-size blobs
        blob = bytes([rank + 1]) * 40
        allb = P.gather_blobs(blob, rank, world)
        blobs_ok = allb == b"".join(bytes([q_ + 1]) * 40 for q_ in range(world))
        q.put((rank, err, all(s == allsch[0] for s in allsch), id_ok and blobs_ok, (vb, ve)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_view_sharded_allreduce_gloo(world):
    from paper_2203_07308_b200 import build as B
    B.build()
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    shards = [r[4] for r in res]
    assert shards[0][0] == 0 and shards[-1][1] == 30 and shards[0][1] == shards[1][0]
    for rank, err, same_sched, uid_ok, _ in res:
        assert err <= 1e-13, err
        assert same_sched and uid_ok


@pytest.mark.parametrize("cfg,gpus", [(4, 2), (4, 8), (5, 8)])
def test_bench_launcher_dry_run(cfg, gpus):
    """`bench.py --gpus N` without torchrun re-launches itself as N ranks
    (torch.distributed.run, 127.0.0.1); --dry-run stops after every rank has
    derived its shard (C4: contiguous views covering all 1440; C5: images
    8r..8r+7 covering all 64) and rank 0 printed them."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--dry-run", "--gpus", str(gpus),
                          "--cfg", str(cfg)], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == gpus and len(line["shards"]) == gpus
    sh = sorted(line["shards"], key=lambda r: r["rank"])
    if cfg == 4:
        assert sh[0]["views"][0] == 0 and sh[-1]["views"][1] == 1440
        assert all(sh[k]["views"][1] == sh[k + 1]["views"][0] for k in range(gpus - 1))
    else:
        assert sorted(i for r in sh for i in r["images"]) == list(range(8 * gpus))
