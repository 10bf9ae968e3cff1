"""GPU <-> oracle parity through the C-ABI (BASELINE north_star tolerances):
hash codes, tables, sketches and stop points bit-exact; returned ids and evaluated sets bit-exact
given identical tables; similarities within 1e-5 absolute (expected bit-equal under R-2)."""

import numpy as np
import pytest

import oracle as O
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_1906_12211_b200 as pfg  # noqa: E402

DEV = torch.device("cuda:0")
SIM_TOL = 1e-5


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


class Case:
    def __init__(self, name, data, q, family, L, seed, strategy=O.INDEPENDENT, pool_bits=3072, M=32, K=24):
        self.name, self.data, self.q = name, data, q
        fam = {O.HP: "simhash", O.FHTCP: "fht_cp", O.CP: "cp"}[family]
        strat = {O.POOL: "pool", O.TENSOR: "tensor"}.get(strategy, "independent")
        self.gpu = pfg.Index(_cuda(data), 0, fam, seed=seed, reps=L, strategy=strat, pool_bits=pool_bits,
                             sketch_words=M if M > 0 else -1, prefix_bits=K)
        self.orc = O.OracleIndex(data, family, L=L, seed=seed, strategy=strategy, pool_bits=pool_bits, M=M, K=K)


@pytest.fixture(scope="module")
def cases():
    out = {}
    d1, q1 = synth.config_data(1, n=3000, nq=64)
    out["hp"] = Case("hp", d1, q1, O.HP, 16, 1)
    d2, q2 = synth.config_data(2, n=20000, nq=100)
    out["fht"] = Case("fht", d2, q2, O.FHTCP, 24, 3)
    d3, q3 = synth.config_data(4, n=4000, nq=40)
    out["hp_pool"] = Case("hp_pool", d3[:, :64].copy(), q3[:, :64].copy(), O.HP, 20, 2, O.POOL, 512)
    out["fht_pool"] = Case("fht_pool", d2[:6000], q2[:50], O.FHTCP, 20, 5, O.POOL, 3072)
    # more repetitions than the eagerly hashed 32: later repetitions are hashed in the kernels
    # (lane groups of max(1, d'/32) lanes per repetition), d' = 128, 64 and 32
    out["fht_long"] = Case("fht_long", d2[:8000], q2[:40], O.FHTCP, 64, 6)
    out["fht_d40"] = Case("fht_d40", d2[:5000, :40].copy(), q2[:30, :40].copy(), O.FHTCP, 48, 7)
    out["fht_d20"] = Case("fht_d20", d2[:5000, :20].copy(), q2[:30, :20].copy(), O.FHTCP, 40, 8)
    # tensoring (Alg. 2): L = 16 tries from 2 x 4 tuples; FHT-CP with K = 32 bits = 4 functions
    out["hp_tensor"] = Case("hp_tensor", d1, q1, O.HP, 16, 11, O.TENSOR)
    out["fht_tensor"] = Case("fht_tensor", d2[:8000], q2[:40], O.FHTCP, 16, 12, O.TENSOR, K=32)
    out["hp_tensor64"] = Case("hp_tensor64", d1, q1[:32], O.HP, 64, 13, O.TENSOR)
    # exact cross-polytope (d = 32: ell = 6, 4 functions per repetition; d = 100: ell = 8)
    out["cp"] = Case("cp", d1, q1, O.CP, 16, 21)
    out["cp_pool"] = Case("cp_pool", d1, q1[:40], O.CP, 16, 22, O.POOL, 600)
    out["cp100"] = Case("cp100", d2[:6000], q2[:40], O.CP, 12, 23)
    # more repetitions than the blind rounds reach: only those are hashed up front, the queries
    # the fused kernel resumes get the rest in bulk
    out["cp48"] = Case("cp48", d1, q1, O.CP, 48, 24)
    return out


ALL = ["hp", "fht", "hp_pool", "fht_pool"]


# ------------------------------------------------------------------ build-side parity
@pytest.mark.parametrize("name", ALL)
def test_build_arrays_bit_exact(cases, name):
    c = cases[name]
    g, o = c.gpu, c.orc
    assert g.reps == o.L and g.ell == o.ell and g.funcs_per_rep == o.c
    assert np.array_equal(g.export_data().view(np.uint32), o.data().view(np.uint32))
    slots = g.export_slots()
    assert np.array_equal(slots, o.slots())
    if o.strategy == O.POOL:
        assert np.array_equal(g.export_pool_sel(), o.pool_sel())
    osk = o.sketches()
    for j in range(o.L):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids), j
        # inline sketch word = the oracle's per-point sketch of this repetition's slot (R-21)
        assert np.array_equal(tab[:, 1], osk[ids, slots[j]]), j
        assert np.array_equal(g.export_prefix(j), o.prefix_table(j)), j


@pytest.mark.parametrize("d", [20, 32, 40, 100, 130, 300, 700])
def test_fht_tables_every_width(d):
    # FHT-CP independent tables at d' = 32 .. 1024 (k_fht_keys: lane groups of max(1, d'/128) lanes,
    # rows staged in shared memory; d' < 32: one warp per row), against the oracle's codes
    rng = np.random.default_rng(d)
    n = 2500 + d
    data = rng.standard_normal((n, d)).astype(np.float32)
    g = pfg.Index(_cuda(data), 0, "fht_cp", seed=d, reps=5)
    o = O.OracleIndex(data, O.FHTCP, L=5, seed=d)
    for j in range(5):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids), j


@pytest.mark.parametrize("d", [3, 16, 33, 100, 150, 256])
def test_exact_cp_tables_and_codes_every_width(d):
    # exact cross-polytope codes on tcgen05 (k_cp_tc: 3xTF32 values, exact chains for near ties;
    # 128 or 256 hyperplane columns) against the oracle's sequential chains: tables and query codes
    rng = np.random.default_rng(100 + d)
    n = 2000 + d
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((300, d)).astype(np.float32)
    g = pfg.Index(_cuda(data), 0, "cp", seed=d, reps=4, cp_draws=200)
    o = O.OracleIndex(data, O.CP, L=4, seed=d, cp_draws=200)
    for j in range(4):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids), j
    gc, _ = g.hash_queries(q)
    oc, _ = o.hash(q)
    assert np.array_equal(gc, oc)


@pytest.mark.parametrize("name", ["fht", "fht_pool"])
def test_cp_table_bit_exact(cases, name):
    c = cases[name]
    assert np.array_equal(c.gpu.export_cp(), c.orc.cp())


@pytest.mark.parametrize("name", ALL)
def test_query_hashing_bit_exact(cases, name):
    c = cases[name]
    gc, gs = c.gpu.hash_queries(c.q)
    oc, osk = c.orc.hash(c.q)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gs, osk)


@pytest.mark.parametrize("name", ["hp", "fht", "hp_pool"])
@pytest.mark.parametrize("recall,rule,per_round", [(0.9, 0, False), (0.5, 1, False), (0.99, 0, True)])
def test_stop_tables_match_oracle_rule(cases, name, recall, rule, per_round):
    # the device stops iff ip_k >= thr[i][j]; thr must be the smallest float where the oracle's
    # direct evaluation of the rule says stop (R-9/R-10)
    c = cases[name]
    if c.orc.strategy == O.POOL and rule == 1:
        return
    thr, tau = c.gpu.stop_tables(recall, stop_rule=rule, per_round=per_round)
    delta = 1.0 - np.float64(np.float32(recall))
    rng = np.random.default_rng(0)
    L = c.orc.L
    for i in rng.integers(1, 25, size=12):
        for j in rng.integers(1, L + 1, size=6):
            t = thr[i - 1, j - 1]
            if per_round and j < L:
                assert np.isinf(t)
                continue
            if np.isinf(t):
                assert not c.orc.should_stop(int(i), int(j), 1.0, delta, rule)
                continue
            assert c.orc.should_stop(int(i), int(j), float(t), delta, rule)
            if t > -1.0:
                prev = np.nextafter(np.float32(t), np.float32(-2))
                assert not c.orc.should_stop(int(i), int(j), float(prev), delta, rule)
    # filter breakpoints: the quantile rule (R-26, default, at this recall target) and the
    # expected-distance rule (R-15)
    _, tau1 = c.gpu.stop_tables(recall, stop_rule=rule, per_round=per_round, tau_rule=1)
    for tb, f in ((tau, lambda ip: O.tau_prob(ip, delta)), (tau1, lambda ip: O.tau(ip))):
        for t in range(64):
            b = tb[t]
            assert f(float(b)) <= t
            if b > -1.0:
                assert f(float(np.nextafter(np.float32(b), np.float32(-2)))) > t


# ------------------------------------------------------------------ search parity
def _compare(c, k, recall, gpu_kw, orc_kw, trace=True):
    gpu_kw = dict(gpu_kw); orc_kw = dict(orc_kw)
    gpu_kw.setdefault("rep_chunk", 8); orc_kw.setdefault("rep_chunk", 8)
    cap = 1 << 14
    ids, sims, st, tr = c.gpu.search(_cuda(c.q), k, recall, stats=True, trace_cap=cap, **gpu_kw)
    ids, sims = ids.cpu().numpy(), sims.cpu().numpy()
    oids, osims, otr, otids = c.orc.search(c.q, k, recall, trace_cap=cap, **orc_kw)
    assert np.array_equal(st["i_stop"], otr[:, 0]), "stop level"
    assert np.array_equal(st["j_stop"], otr[:, 1]), "stop repetition"
    assert np.array_equal(st["emitted"], otr[:, 2].astype(np.uint32)), "emitted"
    assert np.array_equal(st["filtered"], otr[:, 3].astype(np.uint32)), "filtered"
    assert np.array_equal(st["dups"], otr[:, 4].astype(np.uint32)), "dups"
    assert np.array_equal(st["evaluated"], otr[:, 5].astype(np.uint32)), "evaluated"
    if trace:
        for r in range(len(c.q)):
            n = min(cap, otr[r, 5])
            assert set(tr[r, :n].tolist()) == set(otids[r, :n].tolist()), f"evaluated set of query {r}"
    assert np.array_equal(ids, oids), "ids"
    fin = np.isfinite(osims)
    assert np.all(np.abs(sims[fin] - osims[fin]) <= SIM_TOL)
    assert np.array_equal(np.isfinite(sims), fin)
    return st


@pytest.mark.parametrize("name", ALL)
@pytest.mark.parametrize("R", [1, 8, 16])
@pytest.mark.parametrize("recall", [0.5, 0.9, 0.99])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_parity(cases, name, R, recall, engine):
    c = cases[name]
    _compare(c, 10, recall, dict(rep_chunk=R, engine=engine), dict(rep_chunk=R))


@pytest.mark.parametrize("name", ALL + ["fht_long", "fht_d40", "cp"])
@pytest.mark.parametrize("recall", [0.5, 0.9, 0.99])
@pytest.mark.parametrize("rounds", [0, 1, 3])
def test_search_parity_two_pipelines(cases, name, recall, rounds):
    # pipelines = 2: the two halves of the batch as two searches on two streams (pfg.cu
    # pipeline_params), each with its own fused tail
    c = cases[name]
    _compare(c, 10, recall, dict(rep_chunk=16, engine=0, pipelines=2, rounds=rounds), dict(rep_chunk=16))


def test_two_pipelines_equal_one_pipeline():
    # a larger batch (odd nq): two pipelines identical to one
    data, q = synth.config_data(2, n=60000, nq=4999)
    g = pfg.Index(_cuda(data), 0, "fht_cp", seed=5, reps=48)
    res = []
    for pl in (1, 0, 2):
        ids, sims, st = g.search(_cuda(q), 10, 0.9, stats=True, pipelines=pl)
        res.append((ids.cpu().numpy(), sims.cpu().numpy(), st))
    for ids, sims, st in res[1:]:
        assert np.array_equal(ids, res[0][0]) and np.array_equal(sims.view(np.uint32), res[0][1].view(np.uint32))
        for f in st.dtype.names:
            assert np.array_equal(st[f], res[0][2][f]), f


@pytest.mark.parametrize("name", ["hp_tensor", "fht_tensor", "hp_tensor64"])
@pytest.mark.parametrize("recall", [0.5, 0.9, 0.99])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_parity_tensor(cases, name, recall, engine):
    c = cases[name]
    st = _compare(c, 10, recall, dict(engine=engine), dict())
    assert np.all(st["j_stop"][st["i_stop"] > 0] <= int(round(c.orc.L ** 0.5)))   # shells m <= sqrt(L)
    assert np.all((st["i_stop"] % (2 * c.orc.ell)) == 0)                          # depths in steps of two functions


@pytest.mark.parametrize("name", ["hp_tensor", "fht_tensor"])
def test_tensor_build_bit_exact(cases, name):
    c = cases[name]
    g, o = c.gpu, c.orc
    assert np.array_equal(g.export_pool_sel(), o.pool_sel())
    for j in range(o.L):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids), j


@pytest.mark.parametrize("name", ["fht_long", "fht_d40", "fht_d20"])
@pytest.mark.parametrize("recall", [0.9, 0.99])
@pytest.mark.parametrize("engine", [0, 1, 2])
@pytest.mark.parametrize("R", [8, 16])
def test_search_parity_lazy_hashing(cases, name, recall, engine, R):
    # R = 16: round 3 reaches repetition 49, beyond the eager depth: the active queries' codes and
    # ranges of the next repetitions are computed in bulk before it (engine 0)
    c = cases[name]
    st = _compare(c, 10, recall, dict(rep_chunk=R, engine=engine), dict(rep_chunk=R))
    if recall == 0.99:
        assert np.any(st["j_stop"] > 32) or np.any(st["i_stop"] < 24), "no query reached the lazily hashed repetitions"


@pytest.mark.parametrize("rounds", [1, 3, 64])
@pytest.mark.parametrize("engine", [0, 2])
def test_round_engine_handoff_midway(cases, rounds, engine):
    # queries still running after the bulk rounds resume in the fused kernel from the saved state
    for name in ("hp", "fht", "fht_long"):
        _compare(cases[name], 10, 0.99, dict(rep_chunk=4, engine=engine, rounds=rounds), dict(rep_chunk=4))


# ------------------------------------------------------------------ wide queries, device-side loop
# A query whose evaluated set outgrows `wide` ids moves it to a visit-tag array and continues in the
# device-side round loop (a CUDA graph WHILE node).  By default the loop keeps only the wide queries;
# loop_min = 1 with a large loop_max keeps every query still running after the blind rounds.
@pytest.mark.parametrize("name", ["hp", "fht", "hp_pool", "fht_long"])
@pytest.mark.parametrize("wide", [1, 64])
@pytest.mark.parametrize("recall", [0.9, 0.99])
@pytest.mark.parametrize("R", [4, 16])
@pytest.mark.parametrize("keep_all", [False, True])
def test_search_parity_wide(cases, name, wide, recall, R, keep_all):
    loop = dict(loop_min=1, loop_max=1000000) if keep_all else {}
    st = _compare(cases[name], 10, recall, dict(rep_chunk=R, wide=wide, **loop), dict(rep_chunk=R))
    if keep_all or wide == 1:
        assert np.any(st["flags"] & 16), "no query went wide"


@pytest.mark.parametrize("rounds", [1, 2, 5])
@pytest.mark.parametrize("k", [1, 33])
def test_search_parity_loop_and_wide_mixed(cases, rounds, k):
    # the loop keeps all queries; some widen, some stay in the hash set (and may be handed to the
    # fused kernel's second launch)
    for name in ("hp", "fht", "fht_long"):
        _compare(cases[name], k, 0.99, dict(rep_chunk=4, rounds=rounds, wide=200, loop_min=1, loop_max=1000000),
                 dict(rep_chunk=4))


def test_search_parity_wide_beside_fused(cases):
    # the loop keeps only the wide queries (count above loop_max); the others run in the fused
    # kernel launched beside it on the aux stream
    st = _compare(cases["fht"], 10, 0.99, dict(rep_chunk=8, rounds=2, wide=40, loop_max=1), dict(rep_chunk=8))
    assert np.any(st["flags"] & 16) and np.any(~st["flags"] & 16)


def test_search_parity_wide_deferrals(cases):
    # wide tile buffer at its minimum (one chunk's worth): chunks wait for room in later rounds
    for name in ("hp", "fht_long"):
        _compare(cases[name], 10, 0.99, dict(rep_chunk=8, wide=1, loop_min=1, loop_max=1000000, wide_tiles_min=True),
                 dict(rep_chunk=8))


def test_search_parity_wide_arrays_exhausted(cases):
    # one visit-tag array: the first query to widen takes it, the others go to the fused kernel
    st = _compare(cases["fht"], 10, 0.99, dict(rep_chunk=8, wide=16, loop_min=1, wide_arrays=1), dict(rep_chunk=8))
    assert np.sum((st["flags"] & 16) != 0) == 1


@pytest.mark.parametrize("wide", [0, 1])
def test_exhaustive_search_in_the_loop(cases, wide):
    # recall 1: every query reaches the i = 0 linear scan, which runs as wide tiles in the loop
    c = cases["hp"]
    st = _compare(c, 10, 1.0, dict(rep_chunk=8, wide=wide, loop_min=1, loop_max=1000000), dict(rep_chunk=8))
    assert np.all(st["i_stop"] == 0) and np.all(st["flags"] & 16)


@pytest.mark.parametrize("name", ["hp", "fht"])
@pytest.mark.parametrize("kw", [dict(use_filter=False), dict(stop_rule=1), dict(per_round=True),
                                dict(segment=1), dict(segment=5, rep_chunk=3), dict(tau_rule=1),
                                dict(eps=0.2, tau_rule=1), dict(eps=-0.2, tau_rule=1),
                                dict(rep_chunk=32), dict(uniform_chunks=True),
                                dict(uniform_chunks=True, rep_chunk=3, eps=0.1, tau_rule=1)])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_parity_options(cases, name, kw, engine):
    c = cases[name]
    okw = dict(kw)
    _compare(c, 10, 0.9, dict(kw, engine=engine), okw)


def _per_level_emitted(runs, K):
    """emitted positions per (query, level) from searches that differ only in the recall target: with
    the filter off and the stop rule checked once per level (stop_granularity 1) the positions a query
    retrieves down to a level do not depend on the target, so the totals of two runs that stop at
    levels i and i + 1 differ by exactly what level i emitted; level K's count is the total of a run
    that stops there.  runs: [(i_stop[nq], emitted[nq])]; returns {(query, level): count}"""
    nq = len(runs[0][0])
    out = {}
    for r in range(nq):
        tot = {}
        for i_stop, emitted in runs:
            i, e = int(i_stop[r]), int(emitted[r])
            assert tot.setdefault(i, e) == e, "the total at a stop level depends on the recall target"
        for i, e in tot.items():
            if i == K:
                out[(r, i)] = e
            elif i + 1 in tot:
                assert e >= tot[i + 1]
                out[(r, i)] = e - tot[i + 1]
    return out


@pytest.mark.parametrize("name", ["hp", "fht", "hp_pool"])
@pytest.mark.parametrize("engine", [0, 1])
def test_emitted_per_level(cases, name, engine):
    # SURVEY 8(c) parity object "emitted-position count per level", reconstructed on each side from
    # its own totals along a ladder of recall targets and compared cell by cell
    c = cases[name]
    K = 24
    ladder = [0.05, 0.2, 0.35, 0.5, 0.65, 0.8, 0.9, 0.95, 0.98, 0.995, 0.999]
    g_runs, o_runs = [], []
    for recall in ladder:
        _, _, st = c.gpu.search(_cuda(c.q), 10, recall, stats=True, rep_chunk=8, engine=engine, use_filter=False,
                                per_round=True)
        _, _, otr = c.orc.search(c.q, 10, recall, rep_chunk=8, use_filter=False, per_round=True)
        assert np.array_equal(st["j_stop"][st["i_stop"] > 0], np.full(int((st["i_stop"] > 0).sum()), c.orc.L))
        g_runs.append((st["i_stop"].copy(), st["emitted"].copy()))
        o_runs.append((otr[:, 0].copy(), otr[:, 2].astype(np.uint32)))
    g, o = _per_level_emitted(g_runs, K), _per_level_emitted(o_runs, K)
    assert g == o
    levels = {lv for _, lv in g}
    assert len(g) >= len(c.q) and len(levels) >= 3, (len(g), sorted(levels))


@pytest.mark.parametrize("k", [1, 33, 100])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_parity_k(cases, k, engine):
    _compare(cases["fht"], k, 0.9, dict(rep_chunk=8, engine=engine), dict(rep_chunk=8))


def test_exhaustive_recall_one_is_bruteforce(cases):
    # delta = 0: no stop above i = 0; the i = 0 scan returns the exact top-k (R-13)
    c = cases["hp"]
    st = _compare(c, 10, 1.0, dict(rep_chunk=8), dict(rep_chunk=8), trace=False)
    assert np.all(st["i_stop"] == 0)
    ids, _, _ = c.gpu.search(_cuda(c.q), 10, 1.0, stats=True)
    bi, _ = O.bruteforce(c.orc.data(), O.normalize(c.q), 10)
    assert np.array_equal(ids.cpu().numpy(), bi)


def test_k_greater_than_n():
    data, q = synth.config_data(1, n=7, nq=5)
    g = pfg.Index(_cuda(data), 0, "simhash", seed=4, reps=3)
    o = O.OracleIndex(data, O.HP, L=3, seed=4)
    ids, sims, st = g.search(_cuda(q), 12, 0.9, stats=True)
    oids, osims, otr = o.search(q, 12, 0.9, rep_chunk=pfg.DEFAULT_REP_CHUNK)
    assert np.array_equal(ids.cpu().numpy(), oids)
    assert np.all(ids.cpu().numpy()[:, 7:] == -1) and np.all(np.isneginf(sims.cpu().numpy()[:, 7:]))
    assert np.all(st["flags"] & 1)


def test_zero_query_row_reported_and_others_answered(cases):
    c = cases["hp"]
    q = c.q.copy()
    q[3] = 0
    with pytest.raises(pfg.PfgError, match="query row 3") as e:
        c.gpu.search(_cuda(q), 10, 0.9)
    assert e.value.status == 2
    # the other rows still get answered
    ids = torch.empty((len(q), 10), dtype=torch.int64, device=DEV)
    sims = torch.empty((len(q), 10), dtype=torch.float32, device=DEV)
    with pytest.raises(pfg.PfgError):
        c.gpu.search(_cuda(q), 10, 0.9, out=(ids, sims))
    oids, _, _ = c.orc.search(np.delete(q, 3, axis=0), 10, 0.9, rep_chunk=pfg.DEFAULT_REP_CHUNK)
    assert np.array_equal(np.delete(ids.cpu().numpy(), 3, axis=0), oids)
    assert np.all(ids.cpu().numpy()[3] == -1) and np.all(np.isnan(sims.cpu().numpy()[3]))


def test_zero_data_row_rejected():
    data, _ = synth.config_data(1, n=100, nq=1)
    data[42] = 0
    with pytest.raises(pfg.PfgError, match="row 42"):
        pfg.Index(_cuda(data), 0, "simhash", reps=2)


def test_bad_arguments(cases):
    g = cases["hp"].gpu
    q = _cuda(cases["hp"].q)
    for kw in (dict(k=0, recall=0.9), dict(k=300, recall=0.9), dict(k=5, recall=0.0), dict(k=5, recall=1.5)):
        with pytest.raises(pfg.PfgError) as e:
            g.search(q, **kw)
        assert e.value.status == 1
    with pytest.raises(pfg.PfgError, match="rep_chunk"):
        g.search(q, 5, 0.9, rep_chunk=64)


def test_host_buffers_equal_device_buffers(cases):
    # e2e path: numpy in/out goes through the library's H2D/D2H copies, same results
    c = cases["fht"]
    a_ids, a_sims = c.gpu.search(_cuda(c.q), 10, 0.9)
    b_ids, b_sims = c.gpu.search(c.q, 10, 0.9)
    assert isinstance(b_ids, np.ndarray)
    assert np.array_equal(a_ids.cpu().numpy(), b_ids)
    assert np.array_equal(a_sims.cpu().numpy(), b_sims)


def test_repeat_search_is_deterministic(cases):
    # the per-slot bitmaps are returned to zero after every query
    c = cases["fht"]
    r1 = c.gpu.search(_cuda(c.q), 10, 0.99, stats=True)
    r2 = c.gpu.search(_cuda(c.q[::-1].copy()), 10, 0.99, stats=True)
    assert np.array_equal(r1[0].cpu().numpy(), r2[0].cpu().numpy()[::-1])
    assert np.array_equal(r1[2]["evaluated"], r2[2]["evaluated"][::-1])


def test_single_query_and_empty_batch(cases):
    c = cases["hp"]
    ids, sims = c.gpu.search(_cuda(c.q[:1]), 10, 0.9)
    oids, _, _ = c.orc.search(c.q[:1], 10, 0.9, rep_chunk=pfg.DEFAULT_REP_CHUNK)
    assert np.array_equal(ids.cpu().numpy(), oids)
    e_ids, _ = c.gpu.search(_cuda(c.q[:0]), 10, 0.9)
    assert e_ids.shape == (0, 10)


# ------------------------------------------------------------------ sharded mode (one GPU)
def test_sharded_merge_equals_per_shard_oracle():
    # each shard = an index over a contiguous id block with the same seed;
    # merging shard-local top-k equals merging the oracle's per-shard results (P15)
    data, q = synth.config_data(2, n=12000, nq=60)
    world, k = 3, 10
    per = len(data) // world
    g_ids, g_sims, o_ids, o_sims = [], [], [], []
    for r in range(world):
        sl = data[r * per:(r + 1) * per]
        g = pfg.Index(_cuda(sl), 0, "fht_cp", seed=7, reps=12, id_offset=r * per)
        i, s = g.search(_cuda(q), k, 0.9)
        g_ids.append(i); g_sims.append(s)
        o = O.OracleIndex(sl, O.FHTCP, L=12, seed=7)
        oi, os_, _ = o.search(q, k, 0.9, rep_chunk=pfg.DEFAULT_REP_CHUNK)
        o_ids.append(np.where(oi >= 0, oi + r * per, -1)); o_sims.append(os_)
    mi, ms = pfg.merge_topk(torch.stack(g_ids), torch.stack(g_sims))
    ci = np.concatenate(o_ids, axis=1); cs = np.concatenate(o_sims, axis=1)
    ref = np.empty((len(q), k), np.int64)
    for t in range(len(q)):
        order = np.lexsort((ci[t], -cs[t]))[:k]
        ref[t] = ci[t, order]
    assert np.array_equal(mi.cpu().numpy(), ref)


def test_merge_of_bruteforce_shards_is_global_bruteforce():
    # P15: merge(brute force per shard) == global brute force (exact identity)
    rng = np.random.default_rng(5)
    x = O.normalize(rng.standard_normal((3000, 20)))
    q = O.normalize(rng.standard_normal((50, 20)))
    k, world = 7, 4
    per = 3000 // world
    ids, sims = [], []
    for r in range(world):
        bi, bs = O.bruteforce(x[r * per:(r + 1) * per], q, k)
        ids.append(bi + r * per); sims.append(bs.astype(np.float32))
    mi, _ = pfg.merge_topk(_cuda(np.stack(ids)), _cuda(np.stack(sims)))
    gi, _ = O.bruteforce(x, q, k)
    assert np.array_equal(mi.cpu().numpy(), gi)


# ------------------------------------------------------------------ serialisation
@pytest.mark.parametrize("name", ["hp", "fht", "hp_pool", "hp_tensor"])
def test_save_load_roundtrip(cases, name, tmp_path):
    c = cases[name]
    path = str(tmp_path / f"{name}.pfg")
    c.gpu.save(path)
    g2 = pfg.Index.load(path)
    assert g2.info == c.gpu.info
    assert np.array_equal(g2.export_data().view(np.uint32), c.gpu.export_data().view(np.uint32))
    assert np.array_equal(g2.export_slots(), c.gpu.export_slots())
    for j in (0, c.orc.L - 1):
        assert np.array_equal(g2.export_table(j), c.gpu.export_table(j))
        assert np.array_equal(g2.export_prefix(j), c.gpu.export_prefix(j))
    q = _cuda(c.q)
    a = c.gpu.search(q, 10, 0.9, stats=True)
    b = g2.search(q, 10, 0.9, stats=True)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    g2.close()


def test_load_rejects_bad_files(tmp_path):
    with pytest.raises(pfg.PfgError) as e:
        pfg.Index.load(str(tmp_path / "missing.pfg"))
    assert e.value.status == 1
    bad = tmp_path / "bad.pfg"
    bad.write_bytes(b"not an index file at all")
    with pytest.raises(pfg.PfgError) as e:
        pfg.Index.load(str(bad))
    assert e.value.status == 1


def test_load_truncated_file_is_a_short_read(cases, tmp_path):
    path = tmp_path / "full.pfg"
    cases["hp"].gpu.save(str(path))
    raw = path.read_bytes()
    cut = tmp_path / "cut.pfg"
    cut.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(pfg.PfgError) as e:
        pfg.Index.load(str(cut))
    assert e.value.status == 7


# ------------------------------------------------------------------ R-25 int16 storage
class Case16(Case):
    def __init__(self, name, data, q, family, L, seed, strategy=O.INDEPENDENT, pool_bits=3072):
        self.name, self.data, self.q = name, data, q
        fam = "simhash" if family == O.HP else "fht_cp"
        strat = {O.POOL: "pool", O.TENSOR: "tensor"}.get(strategy, "independent")
        self.gpu = pfg.Index(_cuda(data), 0, fam, seed=seed, reps=L, strategy=strat, pool_bits=pool_bits,
                             storage="i16")
        self.orc = O.OracleIndex(data, family, L=L, seed=seed, strategy=strategy, pool_bits=pool_bits,
                                 storage="i16")


@pytest.fixture(scope="module")
def cases16():
    out = {}
    d1, q1 = synth.config_data(1, n=3000, nq=64)
    out["hp"] = Case16("hp", d1, q1, O.HP, 16, 1)
    d2, q2 = synth.config_data(2, n=20000, nq=100)
    out["fht"] = Case16("fht", d2, q2, O.FHTCP, 24, 3)
    d3, q3 = synth.config_data(4, n=4000, nq=40)
    out["hp_pool"] = Case16("hp_pool", d3[:, :64].copy(), q3[:, :64].copy(), O.HP, 20, 2, O.POOL, 512)
    out["fht_long"] = Case16("fht_long", d2[:8000, :40].copy(), q2[:40, :40].copy(), O.FHTCP, 48, 6)
    out["hp_tensor"] = Case16("hp_tensor", d1, q1, O.HP, 16, 11, O.TENSOR)
    return out


@pytest.mark.parametrize("name", ["hp", "fht", "hp_pool", "fht_long", "hp_tensor"])
def test_int16_rows_and_tables_bit_exact(cases16, name):
    c = cases16[name]
    assert np.array_equal(c.gpu.export_data16(), c.orc.data16())
    for j in (0, c.orc.L - 1):
        tab = c.gpu.export_table(j)
        codes, ids = c.orc.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes)
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids)
    # the fp32 rows are kept for the re-rank of the top-k
    assert np.array_equal(c.gpu.export_data().view(np.uint32), c.orc.data().view(np.uint32))


@pytest.mark.parametrize("name", ["hp", "fht", "hp_pool", "fht_long"])
@pytest.mark.parametrize("R", [8, 16])
@pytest.mark.parametrize("recall", [0.5, 0.9, 0.99])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_parity_int16(cases16, name, R, recall, engine):
    _compare(cases16[name], 10, recall, dict(rep_chunk=R, engine=engine), dict(rep_chunk=R))


@pytest.mark.parametrize("name", ["hp", "fht"])
def test_int16_rerank_and_without(cases16, name):
    # the default fp32 re-rank of the fixed-point top-k returns fp32 similarities of the
    # returned ids (within 1e-5 of the fp32 oracle's similarity of the same pair); without it the
    # fixed-point similarities, both equal to the oracle's
    c = cases16[name]
    _compare(c, 10, 0.9, dict(rep_chunk=8, rerank=False), dict(rep_chunk=8, rerank=False))
    ids, sims = c.gpu.search(_cuda(c.q), 10, 0.9, rep_chunk=8)[:2]
    ids, sims = ids.cpu().numpy(), sims.cpu().numpy()
    xn, qn = c.orc.data(), O.normalize(c.q)
    for r in range(len(c.q)):
        for t in range(10):
            if ids[r, t] >= 0:
                assert abs(sims[r, t] - O.sim(qn[r], xn[ids[r, t]])) <= SIM_TOL


@pytest.mark.parametrize("name", ["hp", "fht_long"])
@pytest.mark.parametrize("k", [1, 33])
def test_search_parity_int16_wide_and_k(cases16, name, k):
    _compare(cases16[name], k, 0.99, dict(rep_chunk=8, wide=16, loop_min=1, loop_max=1000000), dict(rep_chunk=8))


@pytest.mark.parametrize("recall", [0.9, 1.0])
def test_search_parity_int16_tensor_and_exhaustive(cases16, recall):
    _compare(cases16["hp_tensor"], 10, recall, dict(), dict(), trace=recall < 1.0)
    _compare(cases16["hp"], 10, recall, dict(rep_chunk=8), dict(rep_chunk=8), trace=recall < 1.0)


def test_int16_save_load(cases16, tmp_path):
    c = cases16["fht"]
    path = str(tmp_path / "i16.pfg")
    c.gpu.save(path)
    g2 = pfg.Index.load(path)
    assert np.array_equal(g2.export_data16(), c.gpu.export_data16())
    q = _cuda(c.q)
    a, b = c.gpu.search(q, 10, 0.9), g2.search(q, 10, 0.9)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])



# ------------------------------------------------------------------ exact cross-polytope family
@pytest.mark.parametrize("name", ["cp", "cp_pool", "cp100"])
def test_cp_exact_build_bit_exact(cases, name):
    c = cases[name]
    g, o = c.gpu, c.orc
    assert np.array_equal(g.export_cp(), o.cp())
    for j in range(o.L):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids), j
    gc, _ = g.hash_queries(c.q)
    oc, _ = o.hash(c.q)
    assert np.array_equal(gc, oc)


@pytest.mark.parametrize("name", ["cp", "cp_pool", "cp100"])
@pytest.mark.parametrize("recall", [0.5, 0.9, 0.99])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_parity_cp_exact(cases, name, recall, engine):
    _compare(cases[name], 10, recall, dict(rep_chunk=8, engine=engine), dict(rep_chunk=8))


# ------------------------------------------------------------------ randomised option sweep
def test_randomised_option_combinations(cases, cases16):
    # 40 seeded random combinations of the search options on the small cases, both engines, with
    # and without the device-side loop / wide queries: every counter, evaluated set and result
    # must equal the oracle's
    import os
    rng = np.random.default_rng(int(os.environ.get("PFG_SWEEP_SEED", 2024)))
    names = ["hp", "fht", "hp_pool", "fht_long", "cp"]
    for it in range(int(os.environ.get("PFG_SWEEP_N", 40))):
        name = names[it % len(names)]
        c = (cases16 if (it % 7 == 3 and name in cases16) else cases)[name]
        R = int(rng.choice([1, 2, 4, 8, 16, 32]))
        kw = dict(rep_chunk=R, segment=int(rng.choice([1, 5, 12, 30])), eps=float(rng.choice([-0.1, 0.0, 0.3])),
                  tau_rule=int(rng.random() < 0.4),
                  uniform_chunks=bool(rng.random() < 0.3), use_filter=bool(rng.random() < 0.85),
                  stop_rule=int(rng.random() < 0.2 and c.orc.strategy == O.INDEPENDENT))
        gk = dict(kw, engine=int(rng.choice([0, 0, 1, 2])), rounds=int(rng.choice([0, 1, 2, 7])),
                  wide=int(rng.choice([0, 0, 1, 40])))
        k = int(rng.choice([1, 5, 10, 33]))
        recall = float(rng.choice([0.5, 0.8, 0.9, 0.97, 0.99]))
        if rng.random() < 0.5:
            gk.update(loop_min=1, loop_max=1000000)
        _compare(c, k, recall, gk, kw)


# ------------------------------------------------------------------ degenerate shapes
@pytest.mark.parametrize("n,d", [(1, 4), (2, 1), (7, 3), (300, 2), (5000, 1), (3000, 300), (2000, 700)])
@pytest.mark.parametrize("family", [O.HP, O.FHTCP])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_tiny_and_degenerate_shapes(n, d, family, engine):
    rng = np.random.default_rng(n * 31 + d)
    data = rng.standard_normal((n, d)).astype(np.float32)
    data[data == 0] = 1.0
    q = rng.standard_normal((17, d)).astype(np.float32)
    q[q == 0] = 1.0
    # duplicate rows and a query equal to a data row
    if n > 3:
        data[3] = data[1]
        q[0] = data[2]
    c = Case("tiny", data, q, family, 6, 5)
    for k in (1, 5, 12):
        for recall in (0.5, 0.95, 1.0):
            _compare(c, k, recall, dict(rep_chunk=4, engine=engine), dict(rep_chunk=4), trace=recall < 1.0)


def test_fuzz_shapes_families_options():
    # seeded random index shapes x families x strategies x storage x search options, each against the
    # oracle (30 cases by default; PFG_FUZZ_N / PFG_FUZZ_SEED for longer runs)
    import os
    rng = np.random.default_rng(int(os.environ.get("PFG_FUZZ_SEED", 99)))
    nfuzz, compared = int(os.environ.get("PFG_FUZZ_N", 30)), 0
    for it in range(nfuzz):
        big = os.environ.get("PFG_FUZZ_BIG") is not None
        n = int(rng.choice([1, 3, 17, 200, 1000, 2500] + ([20000, 60000] if big else [])))
        d = int(rng.choice([1, 2, 5, 16, 33, 64, 100, 130]))
        family = int(rng.choice([O.HP, O.FHTCP, O.CP])) if d <= 128 else int(rng.choice([O.HP, O.FHTCP]))
        strategy = int(rng.choice([O.INDEPENDENT, O.POOL]))
        L = int(rng.integers(1, 13))
        if family == O.HP and rng.random() < 0.2:
            strategy, L = O.TENSOR, int(rng.choice([4, 16]))   # tensoring: L an even power of two
        storage = "i16" if rng.random() < 0.25 else "f32"
        M = int(rng.choice([32, 32, 8, 0]))
        data = rng.standard_normal((n, d)).astype(np.float32)
        data[data == 0] = 0.5
        q = rng.standard_normal((int(rng.integers(1, 400 if big else 40)), d)).astype(np.float32)
        q[q == 0] = 0.5
        fam = {O.HP: "simhash", O.FHTCP: "fht_cp", O.CP: "cp"}[family]
        strat = {O.POOL: "pool", O.TENSOR: "tensor"}.get(strategy, "independent")
        ell = 1 if family == O.HP else 1 + int(np.ceil(np.log2(max(2, 1 << int(np.ceil(np.log2(max(d, 1))))))))
        pool_bits = int(max(2 * 24, 24 * 4) * ell) if strategy == O.POOL else 3072
        try:
            g = pfg.Index(_cuda(data), 0, fam, seed=int(it + 1), reps=L, strategy=strat, pool_bits=pool_bits,
                          sketch_words=M if M > 0 else -1, storage=storage, cp_draws=200)
        except pfg.PfgError:
            continue  # a combination the library rejects by design (e.g. FHT-CP pool too small)
        o = O.OracleIndex(data, family, L=L, seed=int(it + 1), strategy=strategy, pool_bits=pool_bits, M=M,
                          storage=storage, cp_draws=200)
        c = Case.__new__(Case)
        c.name, c.data, c.q, c.gpu, c.orc = f"fuzz{it}", data, q, g, o
        R = int(rng.choice([1, 3, 8, 16]))
        kw = dict(rep_chunk=R, segment=int(rng.choice([1, 12, 40])), use_filter=bool(rng.random() < 0.8),
                  eps=float(rng.choice([0.0, 0.25])), tau_rule=int(rng.random() < 0.4))
        gk = dict(kw, engine=int(rng.choice([0, 0, 1, 2])), rounds=int(rng.choice([0, 1, 3])),
                  wide=int(rng.choice([0, 0, 2])))
        if rng.random() < 0.5:
            gk.update(loop_min=1, loop_max=1000000)
        k = int(rng.choice([1, 4, 10, 33]))
        recall = float(rng.choice([0.5, 0.9, 0.99, 1.0]))
        _compare(c, k, recall, gk, kw, trace=recall < 1.0)
        g.close()
        compared += 1
    print(f"fuzz: {compared} of {nfuzz} cases compared")
    assert compared >= nfuzz // 2



@pytest.mark.parametrize("rounds", [1, 2, 5])
@pytest.mark.parametrize("recall", [0.9, 0.99, 1.0])
def test_search_parity_cp_partial_hashing(cases, rounds, recall):
    c = cases["cp48"]
    _compare(c, 10, recall, dict(rep_chunk=8, rounds=rounds), dict(rep_chunk=8), trace=recall < 1.0)
    _compare(c, 10, recall, dict(rep_chunk=2, rounds=rounds), dict(rep_chunk=2), trace=recall < 1.0)


@pytest.mark.parametrize("engine", [0, 2])
def test_repeat_search_without_sketches(engine):
    # FHT-CP without sketches (M = 0): the side streams and their events exist from the first
    # search on, so the later eager repetitions hashed beside rounds 0/1 are ordered after the
    # normalisation in every search of the same index (advisor finding, round 1)
    d, q = synth.config_data(2, n=6000, nq=40)
    c = Case("fht_m0", d, q, O.FHTCP, 40, 9, M=0)
    for _ in range(3):
        _compare(c, 10, 0.9, dict(rep_chunk=4, engine=engine), dict(rep_chunk=4))


@pytest.mark.parametrize("name,reps", [("hp", None), ("fht", 12), ("fht_long", 20), ("hp_pool", None)])
@pytest.mark.parametrize("engine", [0, 1, 2])
def test_search_with_precomputed_query_hashes(cases, name, reps, engine):
    # SURVEY 8(e) distributed preparation: codes of the first repetitions and the sketches computed
    # separately (pfg_hash_queries_reps) and passed to the search give the same search
    c = cases[name]
    reps = reps or c.orc.L
    codes, sk = c.gpu.hash_queries_reps(_cuda(c.q), reps)
    oc, osk = c.orc.hash(c.q)
    assert np.array_equal(codes.cpu().numpy().view(np.uint32), oc[:, :reps])
    assert np.array_equal(sk.cpu().numpy().view(np.uint64), osk)
    _compare(c, 10, 0.9, dict(rep_chunk=8, engine=engine, ext_codes=codes, ext_sketches=sk), dict(rep_chunk=8))


@pytest.mark.parametrize("name", ["hp", "fht", "fht_long", "hp_pool"])
def test_results_against_plain_order_oracle(cases, name):
    # R-28: the product sums similarities in the R-2 lane-tree order; the oracle can sum them in the
    # plain sequential order of SURVEY 8(c) O-11.  Against it, ids and stop points must agree except
    # where rounding decides: a similarity tie within 1e-6 (the two lists' exact similarities agree
    # rank by rank) or a k-th similarity within 1e-6 of a stop threshold or filter breakpoint.
    c = cases[name]
    ids, sims, st = c.gpu.search(_cuda(c.q), 10, 0.9, stats=True, rep_chunk=8)[:3]
    ids, sims = ids.cpu().numpy(), sims.cpu().numpy()
    oids, osims, otr = c.orc.search(c.q, 10, 0.9, rep_chunk=8, sim_order=1)
    thr, tau = c.gpu.stop_tables(0.9)
    edges = np.concatenate([thr[np.isfinite(thr)].ravel(), tau[:64]])
    xn, qn = c.orc.data().astype(np.float64), O.normalize(c.q).astype(np.float64)
    exc = 0
    for r in range(len(c.q)):
        if np.array_equal(ids[r], oids[r]) and st["i_stop"][r] == otr[r, 0] and st["j_stop"][r] == otr[r, 1]:
            assert np.all(np.abs(sims[r] - osims[r]) <= 2e-6), r
            continue
        exc += 1
        ea = np.sort(xn[ids[r]] @ qn[r])[::-1]
        eb = np.sort(xn[oids[r]] @ qn[r])[::-1]
        tie = np.all(np.abs(ea - eb) <= 1e-6)
        edge = np.min(np.abs(edges - float(osims[r][-1]))) <= 1e-6 or np.min(np.abs(edges - float(sims[r][-1]))) <= 1e-6
        assert tie or edge, (r, ea, eb)
    print(f"{name}: {exc} of {len(c.q)} queries differ from the plain-order oracle (all explained by rounding)")
    assert exc <= max(1, len(c.q) // 50)


def test_sharded_path_over_nccl_world1():
    # the data-sharded mode's collectives on the GPU over NCCL (one rank: this pod has one GPU per
    # call): gather_rows / gather_merge with an explicit world of 1 are copies, so the plumbing
    # (all_gather_into_tensor of the query codes, sketches, ids and sims on device tensors) runs on
    # NCCL with the product's shapes and dtypes, and the sharded search equals the plain one; the
    # 3-shard merge through the all-gathered layout equals the per-shard oracle merge above
    import os
    import socket
    import torch.distributed as dist
    from paper_1906_12211_b200 import sharded
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        data, q = synth.config_data(2, n=12000, nq=64)
        Q = _cuda(q)
        sh = sharded.ShardedIndex(_cuda(data), 0, 0, "fht_cp", seed=7, reps=40)
        reps = sh.prep_reps()
        codes, sk = sharded.distributed_query_hashes(lambda qs: sh.index.hash_queries_reps(qs, reps), Q)
        # the same all-gather the world > 1 path runs, on NCCL
        g_codes = torch.empty_like(codes)
        dist.all_gather_into_tensor(g_codes, codes)
        assert torch.equal(g_codes, codes)
        ids, sims = sh.search(Q, 10, 0.9, distributed_prep=True)
        ids2, sims2 = sh.index.search(Q, 10, 0.9, ext_codes=g_codes, ext_sketches=sk)
        ids3, sims3 = sh.index.search(Q, 10, 0.9)
        assert torch.equal(ids, ids3) and torch.equal(ids2, ids3) and torch.equal(sims2, sims3)
        # gather of per-shard lists through NCCL, then the library's merge
        g_ids = torch.empty((1 * 64, 10), dtype=ids.dtype, device=DEV)
        dist.all_gather_into_tensor(g_ids, ids.contiguous())
        mi, ms = pfg.merge_topk(g_ids.view(1, 64, 10), sims.view(1, 64, 10))
        assert torch.equal(mi, ids) and torch.equal(ms, sims)
        dist.barrier()
    finally:
        dist.destroy_process_group()
