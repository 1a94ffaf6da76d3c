"""The distributed block Wiedemann sequence through the C ABI (SURVEY §8 b, e;
P:457-463): a DISTRIBUTED handle (options.comm) on a P_r x P_c grid of ranks,
rank (i, j) holding row band i of A and column block j of X, the band
iterates all-gathered among the P_r ranks of a block every step.

On the one-GPU test box the ranks are host threads sharing the device
(ffspmv_comm_create_local: the same library code path, the exchange done by
device copies); one rank over a real NCCL communicator runs in
test_dist_nccl.py.  Every result is compared bit-exactly with the oracle
(R20: a distributed result equals the one-GPU result)."""
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


def _run_grid(ff, n, ri, ci, val, m, X, U, L, pr, pc, want_vout=True):
    import torch
    world = pr * pc
    comms = ff.ffspmv_comm_create_local(world)
    out, errs = [None] * world, [None] * world

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                A = ff.ffspmv_create(n, n, ri, ci, val, m, comm=comms[r], dist_rows=pr)
                info = A.info()
                Xd = torch.from_numpy(X.view(np.int32)).cuda()
                Ud = torch.from_numpy(U.view(np.int32)).cuda() if U is not None else None
                S, V = A.sequence(Xd, L, Ud, want_vout=True, stream=st)
                st.synchronize()
                out[r] = (S.cpu().numpy().view(np.uint32), V.cpu().numpy().view(np.uint32), info)
                del A
        except Exception as e:            # reported by the main thread
            errs[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        c.close()
    for e in errs:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("grid", [(1, 1), (2, 1), (1, 2), (2, 2), (3, 1), (4, 1), (1, 3)])
@pytest.mark.parametrize("m", [3, 65521, (1 << 31) - 1])
def test_dist_sequence_grids(ff, oracle_mod, cuda, m, grid):
    pr, pc = grid
    g = synth.rng(17 * pr + 5 * pc + m % 101)
    n = 700
    ri, ci, val = synth.random_coo(g, n, n, 6 * n, m, dup=0.03)
    for k, ku in ((8, 8), (16, 16), (5, 3), (4, 16), (33, 2)):
        X = synth.uniform(g, (n, k), m)
        U = synth.uniform(g, (n, ku), m)
        L = 7
        Sw, Vw = oracle_mod.sequence(n, ri, ci, val, m, X, L, U, want_vout=True)
        res = _run_grid(ff, n, ri, ci, val, m, X, U, L, pr, pc)
        rows = []
        for r, (S, V, info) in enumerate(res):
            assert np.array_equal(S.reshape(Sw.shape), Sw), (grid, k, ku, r)
            assert np.array_equal(V, Vw), (grid, k, ku, r)
            assert info["dist_ranks"] == pr * pc and info["dist_grid_rows"] == pr
            rows.append((info["dist_band_row0"], info["dist_band_rows"]))
        # the bands of column block 0 tile the rows
        band0 = sorted(rows[i * pc] for i in range(pr))
        assert band0[0][0] == 0 and sum(b[1] for b in band0) == n


def test_dist_sequence_edges(ff, oracle_mod, cuda):
    """U = X, L = 1, more column blocks than columns (an empty block), and a
    band with no entries (rows beyond the nonzeros)."""
    m = 65521
    g = synth.rng(99)
    n = 300
    ri, ci, val = synth.random_coo(g, 200, n, 1500, m)      # rows 200..299 empty
    X = synth.uniform(g, (n, 2), m)
    for grid, L in (((1, 3), 5), ((4, 1), 1), ((2, 2), 6)):
        Sw, Vw = oracle_mod.sequence(n, ri, ci, val, m, X, L, None, want_vout=True)
        for S, V, _ in _run_grid(ff, n, ri, ci, val, m, X, None, L, *grid):
            assert np.array_equal(S.reshape(Sw.shape), Sw), grid
            assert np.array_equal(V, Vw), grid


def test_dist_handle_rejects_other_ops(ff, cuda):
    import torch
    comms = ff.ffspmv_comm_create_local(1)
    m = 65521
    ri, ci, val = synth.random_coo(synth.rng(3), 50, 50, 200, m)
    A = ff.ffspmv_create(50, 50, ri, ci, val, m, comm=comms[0])
    x = torch.zeros(50, dtype=torch.int32, device="cuda")
    with pytest.raises(ff.FFSPMVError) as e:
        ff.ffspmv_apply_transpose(A, 1, x, 0, torch.zeros(50, dtype=torch.int32, device="cuda"))
    assert e.value.status == ff.ERR_UNSUPPORTED
    X = torch.zeros((50, 8), dtype=torch.int32, device="cuda")
    Ypad = torch.zeros((50, 12), dtype=torch.int32, device="cuda")[:, :8]
    with pytest.raises(ff.FFSPMVError) as e:              # distributed blocks are contiguous
        ff.ffspmv_apply_block(A, 8, 1, X, 0, Ypad)
    assert e.value.status == ff.ERR_UNSUPPORTED
    with pytest.raises(ff.FFSPMVError) as e:
        ff.ffspmv_create(50, 60, ri, ci, val, m, comm=comms[0])
    assert e.value.status == ff.ERR_NONSQUARE
    del A
    comms[0].close()


def _run_grid_block(ff, n, ri, ci, val, m, X, Y0, alpha, beta, pr, pc):
    """Every rank runs Y <- alpha A X + beta Y (k = X.shape[1]; k = 1 through
    ffspmv_apply) on a distributed handle with the replicated Y0."""
    import torch
    world = pr * pc
    comms = ff.ffspmv_comm_create_local(world)
    out, errs = [None] * world, [None] * world

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                A = ff.ffspmv_create(n, n, ri, ci, val, m, comm=comms[r], dist_rows=pr)
                Xd = torch.from_numpy(np.ascontiguousarray(X).view(np.int32)).cuda()
                Yd = torch.from_numpy(np.ascontiguousarray(Y0).view(np.int32)).cuda()
                if X.shape[1] == 1:
                    ff.ffspmv_apply(A, alpha, Xd.view(-1), beta, Yd.view(-1), stream=st)
                else:
                    ff.ffspmv_apply_block(A, X.shape[1], alpha, Xd, beta, Yd, stream=st)
                st.synchronize()
                out[r] = Yd.cpu().numpy().view(np.uint32)
                del A
        except Exception as e:            # reported by the main thread
            errs[r] = e

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for c in comms:
        c.close()
    for e in errs:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("grid", [(1, 1), (2, 1), (1, 2), (2, 2), (3, 1), (4, 1)])
@pytest.mark.parametrize("m", [3, 65521, (1 << 31) - 1])
def test_dist_apply_block_grids(ff, oracle_mod, cuda, m, grid):
    """Row-sharded single products on a distributed handle (each
    rank its band x column block, then one all-gather): Y on every rank equals
    the oracle's alpha A X + beta Y, for k = 1 (ffspmv_apply), a ragged k and
    the vectorised widths."""
    pr, pc = grid
    g = synth.rng(31 * pr + 7 * pc + m % 97)
    n = 650
    ri, ci, val = synth.random_coo(g, n, n, 7 * n, m, dup=0.03)
    for k in (1, 5, 8, 16):
        X = synth.uniform(g, (n, k), m)
        Y0 = synth.uniform(g, (n, k), m)
        alpha, beta = int(g.integers(0, m)), int(g.integers(0, m))
        want = oracle_mod.apply_block(n, n, ri, ci, val, m, X, Y0, alpha, beta)
        for r, Y in enumerate(_run_grid_block(ff, n, ri, ci, val, m, X, Y0, alpha, beta, pr, pc)):
            assert np.array_equal(Y.reshape(want.shape), want), (grid, k, r)
