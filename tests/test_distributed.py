"""CPU, world_size 2 over gloo: the multi-GPU decomposition reproduces the
single-process result exactly.

Each rank generates its photon share, packs it ([13][stride] words), the
packed shares are all-gathered in rank order (one collective), the cell size
is all-reduced (max), each rank keeps only the photons within the cell of its
band's hit-point box (the rule fppm_gpu_set_photons_packed applies on the
device) and gathers + tests its own band of raster rows.  The oracle stands in for the per-rank device work
(the decomposition logic, not the kernels, is under test here); the per-rank
results, stitched by rows, must equal one single-process run bit for bit.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

W, N, ITERS = 24, 1 << 13, 3
CFG = dict(n_annuli=2, n_sectors=4, alpha_f=0.01, initial_radius=0.05, r_min_base=5e-5,
           samples_per_iteration=N, threads=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from oracle import Oracle
    from paper_2504_04411_b200.distributed import (allgather_packed, global_cell_size, pack_photons,
                                                   photon_share, row_band, share_stride, unpack_photons)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    hp = orc.gen_raster_hitpoints(W)
    r0, r1 = row_band(W, rank, world)
    mine = {k: v[r0 * W:r1 * W] for k, v in hp.items()}
    sess = orc.session(CFG, mine)
    results = []
    for it in range(1, ITERS + 1):
        b, n = photon_share(N, rank, world)
        part = orc.gen_photons(2, 0x5EED, it, b, n)
        local = {"pos": torch.from_numpy(part["pos"]), "normal": torch.from_numpy(part["nrm"]),
                 "wi": torch.from_numpy(part["wi"]), "power": torch.from_numpy(part["pow"]),
                 "depth": torch.from_numpy(part["depth"].view(np.int32))}
        packed = pack_photons(local["pos"], local["normal"], local["wi"], local["power"], local["depth"],
                              share_stride(N, world))
        full = unpack_photons(allgather_packed(packed), [photon_share(N, r, world)[1] for r in range(world)])
        ph = {"pos": full["pos"].numpy(), "nrm": full["normal"].numpy(), "wi": full["wi"].numpy(),
              "pow": full["power"].numpy(), "depth": full["depth"].numpy().view(np.uint32)}
        assert len(ph["pos"]) == N
        cell = global_cell_size(sess.max_radius())
        # cull to the band's hit-point box grown by the cell (order kept)
        lo, hi = mine["pos"].min(0) - cell, mine["pos"].max(0) + cell
        p64 = ph["pos"].astype(np.float64)
        keep = np.all((p64 >= lo) & (p64 <= hi), axis=1)
        ph = {k: v[keep] for k, v in ph.items()}
        if world > 1:
            assert keep.sum() < N  # the band needs fewer than all photons
        out = sess.iterate(it, ph, cell=cell)
        results.append({k: v for k, v in out.items() if k != "times"})
    np.save(os.path.join(outdir, f"rank{rank}.npy"), results, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_decomposition_matches_single_process(port, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    per_rank = [np.load(tmp_path / f"rank{r}.npy", allow_pickle=True) for r in range(world)]
    hp = port.gen_raster_hitpoints(W)
    sess = port.session(CFG, hp)
    for it in range(1, ITERS + 1):
        want = sess.iterate(it, port.gen_photons(2, 0x5EED, it, 0, N))
        for k in want:
            if k == "times":
                continue
            got = np.concatenate([per_rank[r][it - 1][k] for r in range(world)], axis=0)
            assert np.array_equal(got, want[k]), (it, k)


def test_partitions_cover_exactly():
    from paper_2504_04411_b200.distributed import photon_share, row_band
    for world in (1, 2, 3, 4, 8):
        rows = [row_band(512, r, world) for r in range(world)]
        assert rows[0][0] == 0 and rows[-1][1] == 512
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        shares = [photon_share(1 << 22, r, world) for r in range(world)]
        assert sum(c for _, c in shares) == 1 << 22
        assert all(s[0] + s[1] == t[0] for s, t in zip(shares, shares[1:]))


def _worker_b(rank, world, port, outdir):
    """Option B plumbing: reduce-scatter of partial-sum rows to owners and the
    all-gather of owner values, over gloo."""
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from paper_2504_04411_b200.distributed import (allgather_owner_values, owner_slice,
                                                   reduce_scatter_rows)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, stride = 37, 5
    rows = torch.arange(H * stride, dtype=torch.float64).reshape(H, stride) * (rank + 1)
    mine = reduce_scatter_rows(rows, world)
    h0, n = owner_slice(H, rank, world)
    full = allgather_owner_values(mine[:n, 0].clone(), H, world)
    np.save(os.path.join(outdir, f"b{rank}.npy"), {"mine": mine[:n].numpy(), "full": full.numpy(),
                                                    "h0": h0}, allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_option_b_row_exchange(tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_worker_b, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    H, stride = 37, 5
    base = np.arange(H * stride, dtype=np.float64).reshape(H, stride)
    total = base * sum(r + 1 for r in range(world))
    for r in range(world):
        d = np.load(tmp_path / f"b{r}.npy", allow_pickle=True).item()
        n = len(d["mine"])
        assert np.array_equal(d["mine"], total[d["h0"]:d["h0"] + n])
        assert np.array_equal(d["full"], total[:, 0])


def test_owner_slices_cover_exactly():
    from paper_2504_04411_b200.distributed import owner_slice
    for H in (1, 7, 37, 512 * 512):
        for world in (1, 2, 3, 8):
            s = [owner_slice(H, r, world) for r in range(world)]
            assert s[0][0] == 0 and sum(n for _, n in s) == H
            assert all(a[0] + a[1] == b[0] for a, b in zip(s, s[1:]))
