"""2-D SUMMA sharding (tm_sgemm_summa), verified on one
GPU through tm_sgemm_summa_loopback: every grid rank's C block equals the
oracle's block of C = alpha*A*B + beta*C0 at the north_star 1e-5 (the blocks
are the row/column partitions of tm_dist_rows, pinned in tests/test_oracle.py);
panel bytes received = the A panels of the rank's grid row owned by others plus
the B panels of its grid column owned by others.  Host checks (no GPU): the
panel plan tiles K and respects both K partitions."""
import numpy as np
import pytest

import oracle
import seeded_inputs as si

TOL = 1e-5


@pytest.mark.parametrize("k,pr,pc", [(16384, 2, 4), (1100, 3, 2), (10, 2, 3), (1, 4, 4), (4097, 1, 8), (5000, 8, 1)])
def test_panel_plan(k, pr, pc):
    import paper_1804_10694_b200 as tm
    panels = tm.summa_panels(k, pr, pc)
    assert panels[0][0] == 0 and sum(kr for _, kr in panels) == k
    assert all(a + ka == b for (a, ka), (b, _) in zip(panels, panels[1:]))
    assert all(0 < kr <= 2048 for _, kr in panels)
    for parts in (pr, pc):
        blocks = [tm.dist_rows(k, parts, q) for q in range(parts)]
        for k0, kr in panels:  # inside exactly one block of each partition
            assert sum(1 for b0, br in blocks if b0 <= k0 and k0 + kr <= b0 + br) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("pr,pc,m,n,k", [(1, 1, 300, 260, 200), (1, 3, 500, 300, 700), (2, 2, 1061, 300, 1100),
                                         (2, 3, 777, 650, 2500), (3, 2, 130, 1000, 4100), (2, 4, 1024, 2048, 4096),
                                         (4, 2, 3, 90, 70)])
def test_summa_loopback_blocks_match_oracle(pr, pc, m, n, k):
    import torch
    import paper_1804_10694_b200 as tm
    A, B, C0 = si.matrices(m, n, k, seed=70 + pr * 10 + pc)
    R, D = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    P = pr * pc
    As, Bs, Cs, blocks = [], [], [], []
    for r in range(P):
        (r0, rows), (c0, cols), (a0, ka), (b0, kb) = tm.summa_blocks(m, n, k, pr, pc, r)
        blocks.append(((r0, rows), (c0, cols)))
        As.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows, a0:a0 + ka])).cuda())
        Bs.append(torch.from_numpy(np.ascontiguousarray(B[b0:b0 + kb, c0:c0 + cols])).cuda())
        Cs.append(torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows, c0:c0 + cols])).cuda())
    got = tm.sgemm_summa_loopback(pr, pc, m, n, k, As, Bs, Cs, si.ALPHA, si.BETA)
    torch.cuda.synchronize()
    panels = tm.summa_panels(k, pr, pc)
    for r, ((r0, rows), (c0, cols)) in enumerate(blocks):
        C = Cs[r].cpu().numpy()
        if rows and cols:
            e = float(np.max(oracle.normalized_error(C, R[r0:r0 + rows, c0:c0 + cols], D[r0:r0 + rows, c0:c0 + cols])))
            assert e <= TOL, (r, e)
        # message conservation: A panels from the grid row's other owners, B panels from the column's
        i, j = r // pc, r % pc
        lda_p = (max(kr for _, kr in panels) + 3) // 4 * 4
        ldb_p = (cols + 3) // 4 * 4
        exp = 0
        for k0, kr in panels:
            ja = next(q for q in range(pc) if tm.dist_rows(k, pc, q)[0] <= k0 < sum(tm.dist_rows(k, pc, q)))
            ib = next(q for q in range(pr) if tm.dist_rows(k, pr, q)[0] <= k0 < sum(tm.dist_rows(k, pr, q)))
            exp += (rows * lda_p * 4 if ja != j else 0) + (kr * ldb_p * 4 if ib != i else 0)
        assert got[r] == exp, (r, got[r], exp)


@pytest.mark.gpu
def test_summa_loopback_integer_inputs_bit_exact_and_alpha0():
    import torch
    import paper_1804_10694_b200 as tm
    m, n, k, pr, pc = 600, 520, 3000, 2, 3
    A, B, C0 = si.matrices(m, n, k, seed=79, kind="integer")
    R, _ = oracle.sgemm(si.ALPHA, A, B, si.BETA, C0)
    def run(alpha):
        As, Bs, Cs, blocks = [], [], [], []
        for r in range(pr * pc):
            (r0, rows), (c0, cols), (a0, ka), (b0, kb) = tm.summa_blocks(m, n, k, pr, pc, r)
            blocks.append((r0, rows, c0, cols))
            As.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows, a0:a0 + ka])).cuda())
            Bs.append(torch.from_numpy(np.ascontiguousarray(B[b0:b0 + kb, c0:c0 + cols])).cuda())
            Cs.append(torch.from_numpy(np.ascontiguousarray(C0[r0:r0 + rows, c0:c0 + cols])).cuda())
        tm.sgemm_summa_loopback(pr, pc, m, n, k, As, Bs, Cs, alpha, si.BETA)
        torch.cuda.synchronize()
        out = np.zeros((m, n), np.float32)
        for (r0, rows, c0, cols), C in zip(blocks, Cs):
            out[r0:r0 + rows, c0:c0 + cols] = C.cpu().numpy()
        return out
    assert np.array_equal(run(si.ALPHA).astype(np.float64), R)  # integers: exact in TF32, sums < 2^24
    assert np.array_equal(run(0.0), (np.float32(si.BETA) * C0))  # alpha = 0: beta*C, nothing exchanged
