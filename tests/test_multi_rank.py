"""World-size-2 CPU test of the multi-GPU host path (gloo): points sharded in
contiguous blocks with per-point streams keyed by the global index, the per-
increment all-gather of (Σ, C, ‖r‖, status); the gathered result equals a
single-process run bit for bit. Each rank evaluates its shard with the CPU
oracle here (no GPU in this container); on the box the same plumbing carries
the engine's device outputs over NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_02687_b200 import make_paths
from paper_2306_02687_b200.shard import (all_gather_counts, all_gather_outputs, gather_rows, pack_outputs, pad_block,
                                         shard_range, unpack_outputs)

DESK = [("j2", 1.0, 0.3, 0.01, 0.016), ("elastic", 10.0, 0.3)]
P_TOTAL, N_INCR = 11, 6  # 11 points on 2 ranks: unequal blocks (6, 5), padded like the device


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import pyoracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    md = O.Model(8, 6, 40, 5)
    h = O.Hrom(md.G, md.w, md.mat, DESK, md.volume)
    p0, p1 = shard_range(P_TOTAL, rank, world)
    counts = all_gather_counts(p1 - p0)  # fe2_hrom_gather_layout
    per = max(counts)
    E = make_paths(0, 11, p1 - p0, N_INCR, p0=p0)
    r = h.run(E)
    gathered = []
    for k in range(N_INCR):
        blk = pad_block(pack_outputs(r["sigma"][:, k], r["C"][:, k], r["res_norm"][:, k], r["status"][:, k]), per)
        g = all_gather_outputs(torch.from_numpy(blk))
        gathered.append(g.numpy())
    if rank == 0:
        np.save(out_path, np.stack(gathered))
        np.save(out_path + ".counts.npy", np.array(counts))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gather_equals_single_process(tmp_path):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import pyoracle as O

    world = 2
    out = str(tmp_path / "g.npy")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    g = np.load(out)  # (N_INCR, world*per, 14)
    counts = np.load(out + ".counts.npy").tolist()
    assert counts == [6, 5]
    rows = gather_rows(counts)
    pad = np.setdiff1d(np.arange(g.shape[1]), rows)
    assert len(pad) == 1 and (g[:, pad, 13] == -1).all() and np.isnan(g[:, pad, :13]).all()
    md = O.Model(8, 6, 40, 5)
    ref = O.Hrom(md.G, md.w, md.mat, DESK, md.volume).run(make_paths(0, 11, P_TOTAL, N_INCR))
    for k in range(N_INCR):
        u = unpack_outputs(g[k][rows])
        assert np.array_equal(u["sigma"], ref["sigma"][:, k])
        assert np.array_equal(u["C"], ref["C"][:, k])
        assert np.array_equal(u["res_norm"], ref["res_norm"][:, k])
        assert (u["status"] == 0).all()


def test_shard_range_partitions():
    for P in (1, 7, 65536):
        for w in (1, 2, 3, 8):
            r = [shard_range(P, k, w) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == P
            assert all(r[k][1] == r[k + 1][0] for k in range(w - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
