"""Triangular solves with the GPU factor (tcg_solve_*, SURVEY.md §8(f) rank 3:
the IC(k) preconditioner apply). The reference has no solve, so
parity is against the oracle's fixed-order substitution (oracle.c
orc_trisolve) -- bitwise -- and against dense solves where the factor is exact
(complete fill), within 1e-10 relative."""
import numpy as np
import pytest

from conftest import analyzed, bitwise_equal, planned

pytestmark = pytest.mark.gpu

CASES = ["c1", "c5_m0", "s27_16_k2", "grid20_k2_leaf4", "rand_spd_200", "elast6_k1", "c2", "c3", "c4"]


def factored(T, name):
    fz = T.GpuFactorizer(planned(name))
    fz.factor()
    return fz


@pytest.mark.parametrize("name", CASES)
def test_solves_bitwise_equal_oracle(T, oracle, name):
    fz = factored(T, name)
    try:
        vals = fz.download()
        u = planned(name).pattern
        s = T.GpuTriSolve(fz)
        rng = np.random.default_rng(7)
        b = rng.standard_normal(u.nrows)
        for which, fn in ((3, s.apply), (1, s.forward), (2, s.backward)):
            x = fn(b)
            assert bitwise_equal(x, oracle.trisolve(u, vals, b, which)), (name, which)
        st = s.stats()
        assert st.kernel_launches == 1 and st.depth_forward >= 1 and st.depth_backward >= 1
        # the two halves compose: backward(forward(b)) == apply(b)
        assert bitwise_equal(s.backward(s.forward(b)), s.apply(b))
        s.close()
    finally:
        fz.close()


def test_complete_fill_solve_is_a_direct_solve(T):
    # level >= n: U is the exact Cholesky factor of PᵀAP, so apply() solves A x = b
    a = T.generate("random_spd", 150, 60000, 3)
    an = T.analyze(a, level=150)
    plan = T.Plan(an.a_permuted, an.pattern, an.ranges)
    fz = T.GpuFactorizer(plan)
    try:
        fz.factor()
        s = T.GpuTriSolve(fz)
        ap = an.a_permuted
        A = np.zeros((ap.nrows, ap.nrows))
        for i in range(ap.nrows):
            A[i, ap.col_idx[ap.row_ptr[i]:ap.row_ptr[i + 1]]] = ap.values[ap.row_ptr[i]:ap.row_ptr[i + 1]]
        b = np.random.default_rng(1).standard_normal(ap.nrows)
        x = s.apply(b)
        ref = np.linalg.solve(A, b)
        assert np.max(np.abs(x - ref)) / np.max(np.abs(ref)) <= 1e-10
        s.close()
    finally:
        fz.close()


def test_forward_and_backward_residuals_full_size(T, oracle):
    # size-independent properties at C2's full size: Uᵀ y = b and U x = y to rounding
    fz = factored(T, "c2")
    try:
        u = planned("c2").pattern
        vals = fz.download()
        s = T.GpuTriSolve(fz)
        b = np.random.default_rng(3).standard_normal(u.nrows)
        y = s.forward(b)
        x = s.backward(y)
        rows = np.repeat(np.arange(u.nrows), np.diff(u.row_ptr))
        uty = np.zeros(u.nrows)
        np.add.at(uty, u.col_idx, vals * y[rows])      # (Uᵀ y)_j = sum_i U(i,j) y_i
        ux = np.zeros(u.nrows)
        np.add.at(ux, rows, vals * x[u.col_idx])       # (U x)_i = sum_j U(i,j) x_j
        assert np.max(np.abs(uty - b)) <= 1e-12 * np.max(np.abs(b)) * 10
        assert np.max(np.abs(ux - y)) <= 1e-12 * np.max(np.abs(y)) * 10
        s.close()
    finally:
        fz.close()


def test_device_vectors_and_refactorization(T, oracle):
    import torch
    name = "c5_m0"
    fz = factored(T, name)
    try:
        s = T.GpuTriSolve(fz)
        u = planned(name).pattern
        b = np.random.default_rng(5).standard_normal(u.nrows)
        bd = torch.from_numpy(b).cuda()
        xd = torch.empty_like(bd)
        s.apply_device_ptr(bd.data_ptr(), xd.data_ptr(), 3)
        torch.cuda.synchronize()
        assert bitwise_equal(xd.cpu().numpy(), s.apply(b))
        # in place (b and x alias)
        s.apply_device_ptr(bd.data_ptr(), bd.data_ptr(), 3)
        torch.cuda.synchronize()
        assert bitwise_equal(bd.cpu().numpy(), xd.cpu().numpy())
        # a new matrix on the same pattern: the solve reads the new factor
        _, an2 = analyzed("c5_m63")
        fz.set_values(T.init_factor_values(an2.a_permuted, an2.pattern))
        fz.factor()
        vals2 = fz.download()
        assert bitwise_equal(s.apply(b), oracle.trisolve(u, vals2, b, 3))
        s.close()
    finally:
        fz.close()


def test_zero_and_nan_right_hand_sides(T, oracle):
    fz = factored(T, "c1")
    try:
        s = T.GpuTriSolve(fz)
        n = planned("c1").pattern.nrows
        assert np.all(s.apply(np.zeros(n)) == 0.0)
        b = np.ones(n)
        b[17] = np.nan
        x = s.apply(b)  # NaN spreads along the dependences; no stall
        ref = oracle.trisolve(planned("c1").pattern, fz.download(), b, 3)
        assert np.array_equal(np.isnan(x), np.isnan(ref))
        assert bitwise_equal(x[~np.isnan(x)], ref[~np.isnan(ref)])
        with pytest.raises(ValueError):
            s.apply(np.ones(n + 1))
        s.close()
    finally:
        fz.close()


def test_preconditioned_cg_converges_faster(T):
    # the caller the solve exists for: IC(1)-preconditioned CG on C5's matrix
    _, an = analyzed("c5_m0")
    ap = an.a_permuted
    rows = np.repeat(np.arange(ap.nrows), np.diff(ap.row_ptr))

    def matvec(v):
        out = np.zeros(ap.nrows)
        np.add.at(out, rows, ap.values * v[ap.col_idx])
        return out

    fz = factored(T, "c5_m0")
    s = T.GpuTriSolve(fz)
    b = np.ones(ap.nrows)

    def cg(prec, tol=1e-8, maxit=2000):
        x = np.zeros_like(b)
        r = b.copy()
        z = prec(r)
        p = z.copy()
        rz = r @ z
        for it in range(1, maxit + 1):
            q = matvec(p)
            alpha = rz / (p @ q)
            x += alpha * p
            r -= alpha * q
            if np.linalg.norm(r) <= tol * np.linalg.norm(b):
                return x, it
            z = prec(r)
            rz_new = r @ z
            p = z + (rz_new / rz) * p
            rz = rz_new
        return x, maxit

    try:
        x_ic, it_ic = cg(s.apply)
        x_id, it_id = cg(lambda r: r.copy())
        assert np.linalg.norm(matvec(x_ic) - b) <= 1e-7 * np.linalg.norm(b)
        assert it_ic * 2 < it_id, (it_ic, it_id)
    finally:
        s.close()
        fz.close()


def test_spmv_with_the_system_matrix_is_exact(T):
    # y = A x on the device: products summed in column order, as np.add.at does
    import torch
    _, an = analyzed("c5_m0")
    ap = an.a_permuted
    fz = factored(T, "c5_m0")
    try:
        s = T.GpuTriSolve(fz)
        s.set_matrix(ap)
        x = np.random.default_rng(2).standard_normal(ap.nrows)
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        s.spmv_ptr(xd.data_ptr(), yd.data_ptr())
        torch.cuda.synchronize()
        rows = np.repeat(np.arange(ap.nrows), np.diff(ap.row_ptr))
        ref = np.zeros(ap.nrows)
        np.add.at(ref, rows, ap.values * x[ap.col_idx])
        assert bitwise_equal(yd.cpu().numpy(), ref)
        with pytest.raises(ValueError):
            s.set_matrix(T.generate("grid2d", 3, 3))  # wrong size
        s.close()
    finally:
        fz.close()


@pytest.mark.parametrize("name", ["c5_m0", "c2"])
def test_gpu_pcg(T, name):
    # IC(k)-preconditioned CG on the device: converges, in well under half the
    # iterations of plain CG, to a true residual at the tolerance
    _, an = analyzed(name)
    ap = an.a_permuted
    fz = factored(T, name)
    try:
        s = T.GpuTriSolve(fz)
        s.set_matrix(ap)
        b = np.ones(ap.nrows)
        ic = T.pcg(s, b, tol=1e-8, maxit=3000)
        plain = T.pcg(s, b, tol=1e-8, maxit=3000, precondition=False)
        assert ic.converged and plain.converged
        assert ic.iterations * 2 < plain.iterations, (ic.iterations, plain.iterations)
        rows = np.repeat(np.arange(ap.nrows), np.diff(ap.row_ptr))
        res = np.zeros(ap.nrows)
        np.add.at(res, rows, ap.values * ic.x[ap.col_idx])
        assert np.linalg.norm(res - b) <= 2e-8 * np.linalg.norm(b)
        s.close()
    finally:
        fz.close()


def test_gpu_pcg_check_interval_is_invisible(T):
    # the device-side convergence mask: reading the residual history every
    # iteration or every 8 / 64 gives the same iterations and the same x
    _, an = analyzed("c5_m0")
    ap = an.a_permuted
    fz = factored(T, "c5_m0")
    try:
        s = T.GpuTriSolve(fz)
        s.set_matrix(ap)
        b = np.random.default_rng(4).standard_normal(ap.nrows)
        runs = [T.pcg(s, b, tol=1e-9, maxit=500, check_every=c) for c in (1, 8, 64)]
        for r in runs[1:]:
            assert r.converged and r.iterations == runs[0].iterations
            assert r.relative_residual == runs[0].relative_residual
            assert bitwise_equal(r.x, runs[0].x)
        # maxit not a multiple of the interval; not converged
        short = T.pcg(s, b, tol=1e-30, maxit=13, check_every=8)
        assert not short.converged and short.iterations == 13
        with pytest.raises(ValueError):
            T.pcg(s, b, check_every=0)
        s.close()
    finally:
        fz.close()


def test_gpu_pcg_exact_preconditioner_stops_clean(T):
    # complete fill: the apply is a direct solve, r reaches (near) zero at once;
    # the frozen iterations after it must not spoil x
    a = T.generate("random_spd", 120, 40000, 5)
    an = T.analyze(a, level=120)
    fz = T.GpuFactorizer(T.Plan(an.a_permuted, an.pattern, an.ranges))
    try:
        fz.factor()
        s = T.GpuTriSolve(fz)
        s.set_matrix(an.a_permuted)
        b = np.random.default_rng(6).standard_normal(an.a_permuted.nrows)
        res = T.pcg(s, b, tol=1e-8, maxit=50, check_every=16)
        assert res.converged and res.iterations <= 3 and np.all(np.isfinite(res.x))
        zero = T.pcg(s, np.zeros_like(b), tol=1e-8)
        assert zero.converged and zero.iterations == 0
        s.close()
    finally:
        fz.close()


def test_async_apply_matches_and_queues(T):
    # tcg_solve_apply_async: same bits as the synchronous apply; several queued
    # back to back (chained through one buffer) before one tcg_solve_sync
    import torch
    fz = factored(T, "c5_m0")
    try:
        s = T.GpuTriSolve(fz)
        n = planned("c5_m0").pattern.nrows
        b = np.random.default_rng(8).standard_normal(n)
        ref = b.copy()
        for _ in range(4):
            ref = s.apply(ref)
        v = torch.from_numpy(b).cuda()
        torch.cuda.synchronize()
        for _ in range(4):
            s.apply_async_ptr(v.data_ptr(), v.data_ptr(), 3)
        s.sync()
        assert bitwise_equal(v.cpu().numpy(), ref)
        with pytest.raises(ValueError):
            s.apply_async_ptr(v.data_ptr(), v.data_ptr(), 4)
        s.close()
    finally:
        fz.close()
