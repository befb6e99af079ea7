"""GPU parity of K8 (rk_pair.cu, RK_OPT_FUSED_STEP = 3): two chained Runge–Kutta stages per
launch (RK4 = two launches, explicit midpoint = one, Gragg's modified midpoint = one + its last
stage from the written-ahead Y3 and W), the first stage's slope evaluated on the
tile grown by one cell and never stored.  Gate: bitwise equality with the fp64 oracle
(R-17) over several steps, on tile-aligned grids (nx % 32 == 0, ny % 16 == 0) from one
tile to many with ragged z chunks, every z-chunk length (the chunk's two extra stage-A planes and
four raw planes recomputed), the 2-cell periodic margin at every domain edge, and the
stage-by-stage fallback on grids K8 does not take."""
import numpy as np
import pytest

import oracle
import rk_inputs

pytestmark = pytest.mark.gpu
OS = oracle.SCHEMES
PAIR = ["rk4", "midpoint", "modified_midpoint"]
LAUNCHES = {"rk4": 2, "midpoint": 1, "modified_midpoint": 2}  # K8 (+ K3 last stage for Gragg)


@pytest.fixture(scope="module")
def ctx():
    import paper_2309_05331_b200 as rk
    c = rk.Context(0, 1, 0)
    yield c
    c.close()


def bitwise(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def first_mismatch(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
    return (bad.size, bad[:4], a[bad[:4]], b[bad[:4]]) if bad.size else None


def pair_state(ctx, dims, u0, mode=3):
    import paper_2309_05331_b200 as rk
    st = ctx.grid(*dims, 2)
    st.set_rhs_gray_scott()
    st.set(u0)
    st.set_option(rk.OPT_COOP_MAX_CELLS, 0)
    st.set_option(rk.OPT_FUSED_STEP, mode)
    return st


def perturbed_ic(nx, ny, nz, seed=42):
    u0 = rk_inputs.gray_scott_ic(nx, ny, nz, seed=seed)
    return u0 + 0.01 * rk_inputs.random_state(u0.size, 5).reshape(u0.shape)


GRIDS = [(32, 16, 1), (32, 16, 3), (32, 32, 2), (64, 32, 5), (96, 48, 20), (128, 64, 37), (64, 16, 70)]


@pytest.mark.parametrize("scheme", PAIR)
@pytest.mark.parametrize("dims", GRIDS, ids=lambda d: "x".join(map(str, d)))
def test_pair_steps_bitwise(ctx, scheme, dims):
    u0 = perturbed_ic(*dims)
    st = pair_state(ctx, dims, u0)
    p = oracle.gray_scott_problem(*dims)
    u = u0
    before = st.stats()
    for k in range(3):
        st.do_step(scheme, float(k), 1.0)
        u = oracle.step(p, OS[scheme], float(k), 1.0, u)
        got = st.get()
        assert bitwise(got, u), (scheme, dims, k, first_mismatch(got, u))
    launches = st.stats()["stage_launches"] - before["stage_launches"]
    st.close()
    assert launches == 3 * LAUNCHES[scheme]


@pytest.mark.parametrize("pz", [1, 2, 3, 5, 8, 64])
@pytest.mark.parametrize("scheme", PAIR)
def test_pair_zchunks_bitwise(ctx, scheme, pz, monkeypatch):
    monkeypatch.setenv("RKB_PZ", str(pz))
    dims = (64, 32, 23)
    u0 = perturbed_ic(*dims, seed=7)
    st = pair_state(ctx, dims, u0)
    p = oracle.gray_scott_problem(*dims)
    u = u0
    for k in range(2):
        st.do_step(scheme, float(k), 1.0)
        u = oracle.step(p, OS[scheme], float(k), 1.0, u)
    got = st.get()
    st.close()
    assert bitwise(got, u), first_mismatch(got, u)


@pytest.mark.parametrize("scheme", PAIR)
def test_pair_production_size(ctx, scheme):
    """256x256x100 (the production chunking of the other tests), 2 steps, every element."""
    dims = (256, 256, 100)
    u0 = perturbed_ic(*dims)
    p = oracle.gray_scott_problem(*dims)
    want = u0
    for k in range(2):
        want = oracle.step(p, OS[scheme], float(k), 1.0, want)
    st = pair_state(ctx, dims, u0)
    for k in range(2):
        st.do_step(scheme, float(k), 1.0)
    got = st.get()
    st.close()
    assert bitwise(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("dims", [(33, 17, 9), (40, 12, 6), (64, 24, 5)], ids=lambda d: "x".join(map(str, d)))
def test_pair_fallback_unaligned(ctx, dims):
    """Grids K8 does not take run the stage-by-stage kernels under the same option."""
    u0 = perturbed_ic(*dims)
    st = pair_state(ctx, dims, u0)
    p = oracle.gray_scott_problem(*dims)
    st.do_step("rk4", 0.0, 1.0)
    got = st.get()
    launches = st.stats()["stage_launches"]
    st.close()
    assert bitwise(got, oracle.step(p, OS["rk4"], 0.0, 1.0, u0))
    assert launches == 4


def test_pair_integrate_const_and_graph(ctx):
    import paper_2309_05331_b200 as rk
    dims = (64, 32, 16)
    u0 = perturbed_ic(*dims, seed=3)
    p = oracle.gray_scott_problem(*dims)
    want, n = oracle.integrate_const(p, OS["rk4"], u0, 0.0, 5.0, 1.0)
    st = pair_state(ctx, dims, u0)
    assert st.integrate_const("rk4", 0.0, 5.0, 1.0) == n
    assert bitwise(st.get(), want)
    st.set(u0)
    st.set_option(rk.OPT_USE_GRAPH, 1)
    assert st.integrate_const("rk4", 0.0, 5.0, 1.0) == n
    got = st.get()
    st.close()
    assert bitwise(got, want)


# ---- DOPRI5 pairs: the head pair (PAIR_DP_HEAD: stages 2 + 3) and the error-controlled tail
# pair (PAIR_DP_TAIL: stages 6 + 7), one launch each ----------------------------------------
def dp_oracle_try(dims, u0, dt, tol=1e-6):
    p = oracle.gray_scott_problem(*dims)
    un, err = oracle.step(p, OS["dopri5"], 0.0, dt, u0, with_error=True)
    E = oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), dt, tol, tol)
    return un, E


@pytest.mark.parametrize("dims", [(32, 16, 1), (32, 16, 4), (64, 32, 9), (96, 48, 20), (128, 64, 37)],
                         ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("dt", [1.0, 4.0])
def test_dp_tail_pair_try_bitwise(ctx, dims, dt):
    """One try from the IC (k1 = F(u) first): E bitwise, u_new (accepted) every element; k7
    through the next try's FSAL reuse."""
    u0 = perturbed_ic(*dims)
    want, E_o = dp_oracle_try(dims, u0, dt)
    st = pair_state(ctx, dims, u0)
    s0 = st.stats()
    acc, E, _ = st.try_step("dopri5", 0.0, dt, 1e-6, 1e-6)
    s1 = st.stats()
    launches = s1["stage_launches"] - s0["stage_launches"]
    got = st.get()
    assert E == E_o, (E, E_o)
    assert launches == 5  # k1, the head pair (2, 3), stages 4, 5, the tail pair (6, 7)
    assert s1["pair_launches"] - s0["pair_launches"] == 2 and s1["head_launches"] - s0["head_launches"] == 1
    cells = dims[0] * dims[1] * dims[2]
    assert s1["head_bytes"] - s0["head_bytes"] == 4 * 16 * cells  # u, k1 -> k2, k3 (ABI 5)
    assert s1["pair_bytes"] - s0["pair_bytes"] == (4 + 7) * 16 * cells
    assert bitwise(got, want if acc else u0), first_mismatch(got, want if acc else u0)
    if acc:  # the next try starts from k7 (FSAL): compare its E and result too
        want2, E2_o = dp_oracle_try(dims, want, dt)
        acc2, E2, _ = st.try_step("dopri5", dt, dt, 1e-6, 1e-6)
        assert E2 == E2_o
        if acc2:
            assert bitwise(st.get(), want2)
    st.close()


@pytest.mark.parametrize("pz", [1, 2, 3, 7, 64])
def test_dp_tail_pair_zchunks(ctx, pz, monkeypatch):
    monkeypatch.setenv("RKB_PZ", str(pz))
    dims = (64, 32, 23)
    u0 = perturbed_ic(*dims, seed=11)
    want, E_o = dp_oracle_try(dims, u0, 2.0)
    st = pair_state(ctx, dims, u0)
    acc, E, _ = st.try_step("dopri5", 0.0, 2.0, 1e-6, 1e-6)
    got = st.get()
    st.close()
    assert E == E_o
    assert bitwise(got, want if acc else u0)


def test_dp_tail_pair_integrate_adaptive(ctx):
    """The headline call on a tile-aligned grid: counts identical, final state bitwise."""
    dims = (128, 64, 48)
    u0 = perturbed_ic(*dims, seed=7)
    p = oracle.gray_scott_problem(*dims)
    want, a_o, r_o, rc = oracle.integrate_adaptive(p, OS["dopri5"], u0, 0.0, 20.0, 1.0, 1e-6, 1e-6)
    assert rc == 0 and r_o > 0
    st = pair_state(ctx, dims, u0)
    a, r = st.integrate_adaptive("dopri5", 0.0, 20.0, 1.0, 1e-6, 1e-6)
    got = st.get()
    st.close()
    assert (a, r) == (a_o, r_o)
    assert bitwise(got, want), first_mismatch(got, want)


def test_dp_tail_pair_equals_stage_kernels(ctx):
    """Same try sequence with the tail pair (default) and with the stage-by-stage kernels."""
    import paper_2309_05331_b200 as rk
    dims = (96, 32, 30)
    u0 = perturbed_ic(*dims, seed=5)
    res = []
    for mode in (3, 0):
        st = pair_state(ctx, dims, u0, mode)
        seq = [st.try_step("dopri5", 0.5 * k, 0.5 + k, 1e-7, 1e-7) for k in range(4)]
        res.append((seq, st.get()))
        st.close()
    assert res[0][0] == res[1][0]
    assert bitwise(res[0][1], res[1][1])


@pytest.mark.parametrize("dims", [(64, 32, 2), (64, 32, 3), (96, 48, 20)], ids=lambda d: "x".join(map(str, d)))
def test_dp_tail_pair_halo_path(ctx, dims):
    """The tail pair on the multi-GPU slab path, one GPU (RK_OPT_HALO_LOOPBACK: the 2-deep ghost
    planes of Y_6 and 1-deep of W travel through a 1-rank NCCL communicator): tries and an
    adaptive run bitwise equal to the oracle, down to 2-plane slabs."""
    import paper_2309_05331_b200 as rk
    u0 = perturbed_ic(*dims, seed=9)
    want, E_o = dp_oracle_try(dims, u0, 2.0)
    st = pair_state(ctx, dims, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    before = st.stats()
    acc, E, _ = st.try_step("dopri5", 0.0, 2.0, 1e-6, 1e-6)
    after = st.stats()
    assert E == E_o
    assert bitwise(st.get(), want if acc else u0)
    assert after["halo_exchanges"] - before["halo_exchanges"] == 6  # k1, head pair (u, k1), 4, 5, tail
    st.set(u0)
    p = oracle.gray_scott_problem(*dims)
    want2, a_o, r_o, rc = oracle.integrate_adaptive(p, OS["dopri5"], u0, 0.0, 12.0, 1.0, 1e-6, 1e-6)
    a, r = st.integrate_adaptive("dopri5", 0.0, 12.0, 1.0, 1e-6, 1e-6)
    got = st.get()
    st.close()
    assert (a, r) == (a_o, r_o)
    assert bitwise(got, want2), first_mismatch(got, want2)


@pytest.mark.parametrize("scheme", PAIR)
@pytest.mark.parametrize("dims", [(64, 32, 2), (64, 32, 5), (96, 48, 37)], ids=lambda d: "x".join(map(str, d)))
def test_pair_steps_halo_path(ctx, scheme, dims):
    """RK4 / midpoint pairs on the multi-GPU slab path, one GPU (loopback): u's and Y_3's 2-deep
    ghost planes through a 1-rank NCCL communicator, bitwise equal to the oracle."""
    import paper_2309_05331_b200 as rk
    u0 = perturbed_ic(*dims, seed=4)
    st = pair_state(ctx, dims, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    p = oracle.gray_scott_problem(*dims)
    u = u0
    before = st.stats()
    for k in range(3):
        st.do_step(scheme, float(k), 1.0)
        u = oracle.step(p, OS[scheme], float(k), 1.0, u)
        got = st.get()
        assert bitwise(got, u), (scheme, dims, k, first_mismatch(got, u))
    after = st.stats()
    st.close()
    # on the slab Gragg's K3 last stage is an interior and a boundary launch (overlapped halo)
    slab_launches = {"rk4": 2, "midpoint": 1, "modified_midpoint": 3 if dims[2] > 2 else 2}
    assert after["stage_launches"] - before["stage_launches"] == 3 * slab_launches[scheme]
    assert after["halo_exchanges"] - before["halo_exchanges"] == 3 * LAUNCHES[scheme]


def test_pair_max_size_1024_cubed(ctx):
    """Maximum size through K8: a 1024^3 grid (2^31 values per array; u, u_new, Y3, W ~ 69 GiB),
    padded offsets of the upper planes beyond int32.  One RK4 step (two pair launches) and one
    explicit-midpoint step; sampled cells (last planes, periodic corners, the IC cube's faces)
    bitwise against the oracle on their radius-5 neighbourhoods."""
    import gc
    gc.collect()
    n = 1024
    u0 = rk_inputs.gray_scott_ic(n, n, n, seed=42)
    st = pair_state(ctx, (n, n, n), u0)
    before = st.stats()["pair_launches"]
    st.do_step("rk4", 0.0, 1.0)
    g4 = st.get()
    st.set(u0)
    st.do_step("midpoint", 0.0, 1.0)
    g2 = st.get()
    launches = st.stats()["pair_launches"] - before
    st.close()
    assert launches == 3
    lo, hi = rk_inputs.cube_range(n)
    pts = [(1023, 1023, 1023), (1023, 0, 511), (1022, 1023, 0), (0, 0, 0), (lo, lo, lo),
           (hi - 1, hi, lo - 1), (hi, 700, hi - 1), (900, lo + 3, hi), (512, 15, 31), (1, 16, 32)]
    r = 5
    p = oracle.gray_scott_problem(2 * r + 1, 2 * r + 1, 2 * r + 1)
    for (z, y, x) in pts:
        idx = lambda c, m: [(c + d) % m for d in range(-r, r + 1)]  # noqa: E731
        blk = np.ascontiguousarray(u0[np.ix_(idx(z, n), [0, 1], idx(y, n), idx(x, n))])
        w4 = oracle.step(p, OS["rk4"], 0.0, 1.0, blk).reshape(blk.shape)
        w2 = oracle.step(p, OS["midpoint"], 0.0, 1.0, blk).reshape(blk.shape)
        assert bitwise(g4[z, :, y, x], w4[r, :, r, r]), ("rk4", z, y, x)
        assert bitwise(g2[z, :, y, x], w2[r, :, r, r]), ("midpoint", z, y, x)
    del g4, g2, u0
    gc.collect()


def _mixed_sequence(st):
    """Every path that shares a state's k buffers, interleaved: K8 RK4 / midpoint / Gragg pairs
    (Y3, W scratch in k buffers 0, 1), DOPRI5 tries (FSAL k1 in buffer 0, the tail pair's k7 in
    buffer 1), Adams steps, CK54 / RKF78 stage by stage, an adaptive run."""
    out, tries = [], []
    st.do_step("rk4", 0.0, 1.0)
    for k in range(2):
        tries.append(st.try_step("dopri5", 1.0 + k, 0.5, 1e-6, 1e-6))
    st.do_step("rk4", 2.0, 1.0)  # after an accepted FSAL try: k1 must not be reused
    tries.append(st.try_step("dopri5", 3.0, 0.5, 1e-6, 1e-6))
    out.append(st.get())
    st.do_step("ab2", 4.0, 0.5)
    st.do_step("modified_midpoint", 4.5, 0.5)
    tries.append(st.try_step("dopri5", 5.0, 0.5, 1e-6, 1e-6))
    st.do_step("midpoint", 5.5, 0.5)
    tries.append(st.try_step("cash_karp54", 6.0, 0.25, 1e-6, 1e-6))
    st.do_step("rkf78", 6.25, 0.25)
    out.append(st.get())
    tries.append(st.integrate_adaptive("dopri5", 6.5, 9.0, 0.5, 1e-6, 1e-6))
    st.do_step("rk4", 9.0, 1.0)
    out.append(st.get())
    return out, tries


@pytest.mark.parametrize("loopback", [0, 1], ids=["one_gpu", "slab_path"])
def test_pair_mixed_sequence_equals_stage_kernels(ctx, loopback):
    import paper_2309_05331_b200 as rk
    dims = (96, 32, 21)
    u0 = perturbed_ic(*dims, seed=12)
    res = []
    for mode in (3, 0):
        st = pair_state(ctx, dims, u0, mode)
        st.set_option(rk.OPT_HALO_LOOPBACK, loopback)
        res.append(_mixed_sequence(st))
        st.close()
    (g3, t3), (g0, t0) = res
    assert t3 == t0
    for i, (a, b) in enumerate(zip(g3, g0)):
        assert bitwise(a, b), (i, first_mismatch(a, b))


# ---- the head pair (stages 2 + 3) on every tableau that admits it: Cash–Karp 5(4), Dormand–Prince
# fixed step and error-controlled (both ratio readings), RKF 7(8) -------------------------------
HEAD_CASES = [("cash_karp54", 0), ("cash_karp54", 1), ("dopri5", 0), ("rkf78", 0), ("rkf78", 1)]


@pytest.mark.parametrize("dims", [(32, 16, 1), (64, 32, 9), (96, 48, 20)], ids=lambda d: "x".join(map(str, d)))
@pytest.mark.parametrize("case", HEAD_CASES, ids=lambda c: f"{c[0]}-{'try' if c[1] else 'step'}")
def test_head_pair_schemes_bitwise(ctx, case, dims):
    """Stages 2 + 3 as one K8 launch for every eligible tableau: bitwise vs the oracle, one head
    launch per step / try, 4 arrays instead of 7."""
    name, adaptive = case
    u0 = perturbed_ic(*dims, seed=21)
    p = oracle.gray_scott_problem(*dims)
    st = pair_state(ctx, dims, u0)
    s0 = st.stats()
    if adaptive:
        acc, E, _ = st.try_step(name, 0.0, 1.0, 1e-6, 1e-6)
        un, err = oracle.step(p, OS[name], 0.0, 1.0, u0, with_error=True)
        assert E == oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), 1.0, 1e-6, 1e-6)
        want = un if acc else u0
    else:
        st.do_step(name, 0.0, 1.0)
        want = oracle.step(p, OS[name], 0.0, 1.0, u0)
    s1 = st.stats()
    got = st.get()
    st.close()
    assert bitwise(got, want), first_mismatch(got, want)
    assert s1["head_launches"] - s0["head_launches"] == 1
    cells = dims[0] * dims[1] * dims[2]
    assert s1["head_bytes"] - s0["head_bytes"] == 4 * 16 * cells
    if not adaptive:  # + the fixed-step tail pair (stages L-1, L after the write-ahead stage L-2)
        assert s1["pair_launches"] - s0["pair_launches"] == 2
        if name in ("cash_karp54", "dopri5"):  # k1 2 + head 4 + stage 4 (Y5, Z6, W) 7 + tail 4
            assert s1["stage_bytes"] - s0["stage_bytes"] == 17 * 16 * cells


@pytest.mark.parametrize("name", ["cash_karp54", "rkf78"])
def test_head_pair_integrate_adaptive_counts(ctx, name):
    """A whole error-controlled integration with the head pair in every try: accepted / rejected
    counts identical to the oracle's, final state bitwise."""
    dims = (64, 32, 12)
    u0 = perturbed_ic(*dims, seed=8)
    p = oracle.gray_scott_problem(*dims)
    want, a_o, r_o, rc = oracle.integrate_adaptive(p, OS[name], u0, 0.0, 10.0, 1.0, 1e-6, 1e-6)
    assert rc == 0
    st = pair_state(ctx, dims, u0)
    a, r = st.integrate_adaptive(name, 0.0, 10.0, 1.0, 1e-6, 1e-6)
    got = st.get()
    heads = st.stats()["head_launches"]
    st.close()
    assert (a, r) == (a_o, r_o)
    assert heads == a + r
    assert bitwise(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("dims", [(64, 32, 2), (64, 32, 7)], ids=lambda d: "x".join(map(str, d)))
def test_head_pair_halo_path_ck54(ctx, dims):
    """The head pair on the slab path (one-GPU loopback through the 1-rank NCCL communicator):
    u's and k1's two boundary planes each side exchanged before the launch; bitwise."""
    import paper_2309_05331_b200 as rk
    u0 = perturbed_ic(*dims, seed=5)
    p = oracle.gray_scott_problem(*dims)
    un, err = oracle.step(p, OS["cash_karp54"], 0.0, 2.0, u0, with_error=True)
    E_o = oracle.error_ratio_max(err, u0, oracle.rhs(p, u0), 2.0, 1e-6, 1e-6)
    st = pair_state(ctx, dims, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    acc, E, _ = st.try_step("cash_karp54", 0.0, 2.0, 1e-6, 1e-6)
    heads = st.stats()["head_launches"]
    got = st.get()
    st.close()
    assert E == E_o
    assert heads == 1
    assert bitwise(got, un if acc else u0), first_mismatch(got, un if acc else u0)


@pytest.mark.parametrize("name", ["cash_karp54", "dopri5", "rkf78"])
@pytest.mark.parametrize("dims", [(64, 32, 2), (64, 32, 7)], ids=lambda d: "x".join(map(str, d)))
def test_fixed_tail_pair_halo_path(ctx, name, dims):
    """The fixed-step tail pair on the slab path (one-GPU loopback, 1-rank NCCL): Y_{L-1}'s two
    boundary planes and Z_L's one exchanged before the launch; three steps bitwise."""
    import paper_2309_05331_b200 as rk
    u0 = perturbed_ic(*dims, seed=6)
    p = oracle.gray_scott_problem(*dims)
    want = u0
    for m in range(3):
        want = oracle.step(p, OS[name], float(m), 0.5, want)
    st = pair_state(ctx, dims, u0)
    st.set_option(rk.OPT_HALO_LOOPBACK, 1)
    s0 = st.stats()
    for m in range(3):
        st.do_step(name, float(m), 0.5)
    s1 = st.stats()
    got = st.get()
    st.close()
    assert s1["pair_launches"] - s0["pair_launches"] == 6  # head + tail per step
    assert bitwise(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("name", ["cash_karp54", "dopri5", "rkf78"])
def test_fixed_tail_pair_integrate_const(ctx, name):
    """integrate_const (several steps, CUDA-graph replay on) through the head and tail pairs,
    bitwise against the oracle's steps."""
    import paper_2309_05331_b200 as rk
    dims = (96, 48, 20)
    u0 = perturbed_ic(*dims, seed=9)
    p = oracle.gray_scott_problem(*dims)
    want, n_o = oracle.integrate_const(p, OS[name], u0, 0.0, 3.0, 0.5)
    st = pair_state(ctx, dims, u0)
    st.set_option(rk.OPT_USE_GRAPH, 1)
    assert st.integrate_const(name, 0.0, 3.0, 0.5) == n_o
    got = st.get()
    st.close()
    assert bitwise(got, want), first_mismatch(got, want)
