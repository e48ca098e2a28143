"""Multi-process (gloo, world size 2) CPU tests of the H-sharded exchange
protocol used by icnnm_sharded_solve.

The GPU test suite runs the product's sharded kernels with virtual slabs on one
device; these tests run the same protocol -- the library's shard plan, the
forward halo shift of the last kh-1 rows to the next rank, the reverse
halo-add of adjoint partial sums, and ONE all-reduce of [norm^2 (k) | report
scalars] per iteration -- across two real processes, on a restated numpy
iteration, and check that it equals the unsharded iteration.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _forward_slab(Lext, K, ks):
    """A(L~)K on slab rows given L~ with kh-1 halo rows first (non-periodic in
    H, periodic in W, T): row h of the slab reads Lext[h + kh-1 - sh]."""
    kh, kw, kt = ks
    rows = Lext.shape[0] - (kh - 1)
    cols = []
    for sh in range(kh):
        for sw in range(kw):
            for st in range(kt):
                sl = Lext[kh - 1 - sh: kh - 1 - sh + rows]
                cols.append(np.roll(sl, (sw, st), axis=(1, 2)).ravel())
    A = np.stack(cols, axis=1)
    return A @ K


def _adjoint_slab(U, ks, rows, W, T):
    """out[i] += U[i + s, s] for slab rows i+s; returns kh-1 halo rows + rows."""
    kh, kw, kt = ks
    out = np.zeros((rows + kh - 1, W, T))
    col = 0
    for sh in range(kh):
        for sw in range(kw):
            for st in range(kt):
                u = U[:, col].reshape(rows, W, T)
                out[kh - 1 - sh: kh - 1 - sh + rows] += np.roll(u, (-sw, -st), axis=(1, 2))
                col += 1
    return out


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, ROOT)
        import paper_2604_17001_b200 as P
        from oracle import icnnm_oracle as O

        H, Wd, T, ks = 12, 6, 5, (3, 2, 2)
        k = int(np.prod(ks))
        rng = np.random.default_rng(0)
        X = rng.uniform(0, 1, (H, Wd, T))
        mask = (rng.uniform(0, 1, X.shape) < 0.5).astype(float)
        B = O.learn_ensemble_basis([rng.uniform(0, 1, X.shape)], ks)
        K = B.K
        row0, rows = P.shard_plan(H, world, ks[0], rank)
        prev, nxt = (rank - 1) % world, (rank + 1) % world

        def shift_forward(last):          # send my last kh-1 rows to rank+1
            recv = torch.empty_like(torch.from_numpy(last))
            reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(last)), nxt),
                    dist.irecv(recv, prev)]
            for r in reqs:
                r.wait()
            return recv.numpy()

        def shift_backward(first):        # send my halo partials to rank-1
            recv = torch.empty_like(torch.from_numpy(first))
            reqs = [dist.isend(torch.from_numpy(np.ascontiguousarray(first)), prev),
                    dist.irecv(recv, nxt)]
            for r in reqs:
                r.wait()
            return recv.numpy()

        # --- halo shift delivers the periodic rows preceding the slab ---
        own = X[row0: row0 + rows]
        halo = shift_forward(own[rows - (ks[0] - 1):])
        expect = X[np.arange(row0 - (ks[0] - 1), row0) % H]
        assert np.array_equal(halo, expect)

        # --- sharded restated iteration vs unsharded (3 iterations) ---
        lam, iters = 1000.0, 3
        pm_full = X * mask
        theta = [min(1e-2 * np.abs(pm_full).max() * k, 1e10)]
        for _ in range(iters):
            theta.append(min(theta[-1] * 1.05, 1e10))

        def unsharded():
            L = pm_full.copy()
            Wm = np.stack([O.circular_shift(L, s).ravel() for s in O.kernel_offsets(ks)], 1) @ K
            for it in range(iters):
                t, r = theta[it], theta[it] / theta[it + 1]
                n = np.linalg.norm(Wm, axis=0)
                c = np.where(n > 1 / t, (1 / t) / np.where(n > 0, n, 1), 1.0)
                adj = O.conv_adjoint((Wm * c) @ K.T, ks, X.shape)
                d = (lam * (pm_full - mask * L) - (t / k) * adj) / (lam * mask + t)
                Lt = L + d + r * d
                L = L + d
                A = np.stack([O.circular_shift(Lt, s).ravel() for s in O.kernel_offsets(ks)], 1)
                Wm = A @ K + r * c * Wm
            return L

        pm = pm_full[row0: row0 + rows]
        mk = mask[row0: row0 + rows]
        L = pm.copy()
        Lext = np.concatenate([shift_forward(L[rows - (ks[0] - 1):]), L], axis=0)
        Wm = _forward_slab(Lext, K, ks)
        for it in range(iters):
            t, r = theta[it], theta[it] / theta[it + 1]
            red = torch.from_numpy(np.concatenate([np.sum(Wm ** 2, axis=0), np.zeros(8)]))
            dist.all_reduce(red)                       # ONE all-reduce per iteration
            n = np.sqrt(red.numpy()[:k])
            c = np.where(n > 1 / t, (1 / t) / np.where(n > 0, n, 1), 1.0)
            part = _adjoint_slab((Wm * c) @ K.T, ks, rows, Wd, T)
            recv = shift_backward(part[: ks[0] - 1])   # reverse halo-add
            adj = part[ks[0] - 1:]
            adj[rows - (ks[0] - 1):] += recv
            d = (lam * (pm - mk * L) - (t / k) * adj) / (lam * mk + t)
            Lt = L + d + r * d
            L = L + d
            Lext = np.concatenate([shift_forward(Lt[rows - (ks[0] - 1):]), Lt], axis=0)
            Wm = _forward_slab(Lext, K, ks) + r * c * Wm
        ref = unsharded()[row0: row0 + rows]
        err = float(np.max(np.abs(L - ref)))
        assert err < 1e-10, err
        q.put((rank, "ok", err))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_protocol_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, info in results:
        assert status == "ok", f"rank {rank}: {info}"


def test_shard_plan_neighbours_cover_ring():
    import paper_2604_17001_b200 as P
    H, G, kh = 64, 4, 9
    plans = [P.shard_plan(H, G, kh, g) for g in range(G)]
    for g, (s, c) in enumerate(plans):
        ps, pc = plans[(g - 1) % G]
        # the kh-1 halo rows of slab g are the last kh-1 rows of slab g-1 (periodic)
        halo_rows = [(s - i) % H for i in range(kh - 1, 0, -1)]
        prev_last = [(ps + pc - i) % H for i in range(kh - 1, 0, -1)]
        assert halo_rows == prev_last
