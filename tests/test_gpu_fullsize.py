"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times:
config 1 completely, config 2 (1M x 100, FHT cross-polytope, 4 GiB budget -> L = 241) on sampled
outputs the oracle computes one by one -- three whole repetition tables, the normalised data, and
the complete searches of 200 queries (the oracle builds only the repetitions they touch); configs
3, 4 and 6 (1M x 300 planted, 1M x 960 pooled with k = 100, the paper's SYNTHETIC set) in two parts:
the configured index with the normalised data, slots, pool selections, (config 3) two whole tables,
every query's codes and sketches and the properties of every query's result; then, on an index of
the same 1M points with 48 repetitions (pooled: a 768-bit pool, 8 sketch words -- what the plain-C
oracle can hash within the suite's time limit), two whole tables and the complete searches of 16
(8) sampled queries element by element."""
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


def _search_equal(g_res, o_res, cap):
    ids, sims, st, tr = g_res
    oids, osims, otr, otids = o_res
    ids, sims = ids.cpu().numpy(), sims.cpu().numpy()
    for col, name in enumerate(["i_stop", "j_stop", "emitted", "filtered", "dups", "evaluated"]):
        assert np.array_equal(st[name].astype(np.int64), otr[:, col].astype(np.int64)), name
    for r in range(len(ids)):
        n = min(cap, otr[r, 5])
        assert set(tr[r, :n].tolist()) == set(otids[r, :n].tolist()), r
    assert np.array_equal(ids, oids)
    assert np.max(np.abs(sims - osims)) <= 1e-5


def test_config1_full():
    c = synth.CONFIGS[1]
    data, q = synth.config_data(1)
    g = pfg.Index(torch.from_numpy(data).to(DEV), 0, "simhash", seed=1, reps=c["reps"])
    o = O.OracleIndex(data, O.HP, L=c["reps"], seed=1)
    cap = 10000
    gr = g.search(torch.from_numpy(q).to(DEV), c["k"], c["recall"], stats=True, trace_cap=cap)
    orr = o.search(q, c["k"], c["recall"], rep_chunk=pfg.DEFAULT_REP_CHUNK, trace_cap=cap)
    _search_equal(gr, orr, cap)
    for j in range(c["reps"]):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes)
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids)


def test_config2_full_sampled():
    c = synth.CONFIGS[2]
    data, q = synth.config_data(2)
    g = pfg.Index(torch.from_numpy(data).to(DEV), c["budget"], "fht_cp", seed=1)
    L = g.info["reps"]
    assert L == pfg.derive_reps(c["n"], c["d"], "fht_cp", c["budget"])[0]
    o = O.OracleIndex(data, O.FHTCP, L=L, seed=1, lazy=True)
    assert np.array_equal(g.export_data().view(np.uint32), o.data().view(np.uint32))
    assert np.array_equal(g.export_slots(), o.slots())
    assert np.array_equal(g.export_cp(), o.cp())
    osk = o.sketches()
    slots = o.slots()
    for j in (0, L // 2, L - 1):
        tab = g.export_table(j)
        codes, ids = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), ids), j
        assert np.array_equal(tab[:, 1], osk[ids, slots[j]]), j
        assert np.array_equal(g.export_prefix(j), o.prefix_table(j)), j
    # the bench's launch: all 10 000 queries in one call; compare a sample of 200 (every 50th)
    cap = 1 << 13
    ids, sims, st, tr = g.search(torch.from_numpy(q).to(DEV), c["k"], c["recall"], stats=True, trace_cap=cap)
    # two round pipelines equal one pipeline (the default)
    ids1, sims1, st1 = g.search(torch.from_numpy(q).to(DEV), c["k"], c["recall"], stats=True, pipelines=2)
    assert torch.equal(ids1, ids) and torch.equal(sims1, sims) and np.array_equal(st1, st)
    sel = np.arange(0, len(q), 50)
    sub = (ids[sel], sims[sel], st[sel], tr[sel])
    orr = o.search(q[sel], c["k"], c["recall"], rep_chunk=pfg.DEFAULT_REP_CHUNK, trace_cap=cap, threads=1)
    _search_equal(sub, orr, cap)


# ------------------------------------------------------------------ configs 3 and 4 at full size
def _truth(x_dev, q_dev, k):
    """exact top-k sims by fp32 inner products on the GPU (torch, TF32 off; test infrastructure)"""
    torch.backends.cuda.matmul.allow_tf32 = False
    x_dev = x_dev / x_dev.norm(dim=1, keepdim=True)
    q_dev = q_dev / q_dev.norm(dim=1, keepdim=True)
    kth = []
    for s in range(0, q_dev.shape[0], 512):
        S = q_dev[s:s + 512] @ x_dev.T
        kth.append(torch.topk(S, k, dim=1).values[:, -1])
    return torch.cat(kth)


def _properties(g, o, data_n, q, k, recall, ids, sims, st):
    """checks that hold at any size: ids distinct and in range, order (sim desc, id asc), every
    returned similarity equal to the oracle's R-2 similarity of that id, the stop decision equal to
    the oracle's stop rule at the returned k-th similarity, recall against the exact top-k"""
    xn = O.normalize(data_n)
    qn = O.normalize(q)
    delta = 1.0 - float(np.float32(recall))
    for r in range(len(q)):
        row, srow = ids[r], sims[r]
        assert np.all(row >= 0) and np.all(row < len(xn)) and len(set(row.tolist())) == k, r
        for t in range(k):
            assert srow[t] == np.float32(O.sim(qn[r], xn[row[t]])), (r, t)
            if t:
                assert srow[t - 1] > srow[t] or (srow[t - 1] == srow[t] and row[t - 1] < row[t]), (r, t)
        i, j = int(st["i_stop"][r]), int(st["j_stop"][r])
        if i > 0:
            ip = float(min(max(srow[k - 1], -1.0), 1.0))
            assert o.should_stop(i, j, ip, delta), (r, i, j)


def _recall(x_t, q_t, ids, k):
    kth = _truth(x_t, q_t, k).cpu().numpy()
    xn = x_t / x_t.norm(dim=1, keepdim=True)
    qn = q_t / q_t.norm(dim=1, keepdim=True)
    ex = torch.einsum("qd,qkd->qk", qn, xn[torch.from_numpy(ids).to(DEV)]).cpu().numpy()
    return float(np.mean(ex >= kth[:, None] - 1e-5))


# reduced index of the element-wise comparison at n = 1M (the oracle hashes every point for every
# repetition / pool function and sketch word it needs, in plain C: the configured L = 458 / 830 / 459
# repetitions, 3 072 pool bits and 32 sketch words cost 4-5 Tflop per config, most of a 20-minute
# suite): 48 repetitions (beyond the eager hashing depth and the third round), for the pooled
# configs a 768-bit pool and 8 sketch words
_REDUCED = {3: dict(reps=48), 4: dict(reps=48, pool_bits=768, sketch_words=8), 6: dict(reps=48, pool_bits=768, sketch_words=8)}


@pytest.mark.parametrize("cfg", [3, 4, 6])
def test_config34_full(cfg):
    c = synth.CONFIGS[cfg]
    data, q = synth.config_data(cfg)
    x_t = torch.from_numpy(data).to(DEV)
    q_t = torch.from_numpy(q).to(DEV)
    strat = O.POOL if c["strategy"] == "pool" else O.INDEPENDENT
    fam = {"simhash": O.HP, "fht_cp": O.FHTCP, "cp": O.CP}[c["family"]]
    pooled = strat == O.POOL

    # ---- part A: the configured index (budget -> L), the launch bench.py times
    g = pfg.Index(x_t, c["budget"], c["family"], seed=1, strategy=c["strategy"])
    L = g.info["reps"]
    assert L == pfg.derive_reps(c["n"], c["d"], c["family"], c["budget"], strategy=c["strategy"])[0]
    # the functions (slots, pool selections, query codes and sketches, the stop rule) do not depend on
    # the data: for the pooled configs the oracle of part A holds the first 2 000 points only (its
    # tables are not used); the independent config 3 builds the two tables compared below lazily
    o = O.OracleIndex(data if not pooled else data[:2000], fam, L=L, seed=1, strategy=strat, lazy=True)
    xn = O.normalize(data)
    assert np.array_equal(g.export_data().view(np.uint32), xn.view(np.uint32))
    assert np.array_equal(g.export_slots(), o.slots())
    if pooled:
        assert np.array_equal(g.export_pool_sel(), o.pool_sel())
    else:
        osk = o.sketches()
        slots = o.slots()
        for j in (0, L - 1):
            tab = g.export_table(j)
            codes, oid = o.rep(j)
            assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
            assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), oid), j
            assert np.array_equal(tab[:, 1], osk[oid, slots[j]]), j
            assert np.array_equal(g.export_prefix(j), o.prefix_table(j)), j
    # query side: codes and sketches of every query bit-exact
    gc, gs = g.hash_queries(q)
    oc, os_ = o.hash(q)
    assert np.array_equal(gc, oc) and np.array_equal(gs, os_)
    # the bench's launch (all queries, default engine): properties at full size
    ids, sims, st = g.search(q_t, c["k"], c["recall"], stats=True)
    ids, sims = ids.cpu().numpy(), sims.cpu().numpy()
    _properties(g, o, data, q, c["k"], c["recall"], ids, sims, st)
    assert _recall(x_t, q_t, ids, c["k"]) >= c["recall"]
    # batch independence + the top-k is exactly the best k of the evaluated set (sampled queries)
    sel = np.arange(0, len(q), max(1, len(q) // 16))
    cap = 1 << 15
    sids, ssims, sst, tr = g.search(torch.from_numpy(q[sel]).to(DEV), c["k"], c["recall"], stats=True, trace_cap=cap)
    assert np.array_equal(sids.cpu().numpy(), ids[sel]) and np.array_equal(sst["j_stop"], st["j_stop"][sel])
    qn = O.normalize(q[sel])
    for r in range(len(sel)):
        ev = tr[r, :min(cap, int(sst["evaluated"][r]))]
        assert len(set(ev.tolist())) == len(ev)
        if sst["evaluated"][r] <= cap:
            sv = np.array([O.sim(qn[r], xn[e]) for e in ev], np.float32)
            order = np.lexsort((ev, -sv))[:c["k"]]
            assert np.array_equal(ev[order].astype(np.int64), ids[sel[r]]), r
    del g, o

    # ---- part B: element by element against the oracle at n = 1M on the reduced index (_REDUCED):
    # two whole tables with their inline sketch words and prefix tables, then the complete searches
    # of 16 sampled queries (8 for config 6, whose queries evaluate most of the points): counters,
    # stop points, evaluated sets, ids, similarities.  With 48 repetitions the queries descend
    # further than under the configured L (more levels, the bitmap / visit-tag modes, k = 100)
    rd = _REDUCED[cfg]
    Lb, pb, Mb = rd["reps"], rd.get("pool_bits", 3072), rd.get("sketch_words", 32)
    g = pfg.Index(x_t, 0, c["family"], seed=1, strategy=c["strategy"], reps=Lb, pool_bits=pb, sketch_words=Mb)
    o = O.OracleIndex(data, fam, L=Lb, seed=1, strategy=strat, pool_bits=pb, M=Mb)
    osk = o.sketches()
    slots = o.slots()
    for j in (0, Lb - 1):
        tab = g.export_table(j)
        codes, oid = o.rep(j)
        assert np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes), j
        assert np.array_equal((tab[:, 0] & np.uint64(0xFFFFFFFF)).astype(np.uint32), oid), j
        assert np.array_equal(tab[:, 1], osk[oid, slots[j]]), j
        assert np.array_equal(g.export_prefix(j), o.prefix_table(j)), j
    esel = sel if cfg != 6 else sel[::2]
    gres = g.search(torch.from_numpy(q[esel]).to(DEV), c["k"], c["recall"], stats=True, trace_cap=cap)
    orr = o.search(q[esel], c["k"], c["recall"], rep_chunk=pfg.DEFAULT_REP_CHUNK, trace_cap=cap, threads=8)
    _search_equal(gres, orr, cap)
    # the same queries inside the whole batch (the bench's launch shape): identical results
    ids_b, sims_b, st_b = g.search(q_t, c["k"], c["recall"], stats=True)
    assert np.array_equal(ids_b.cpu().numpy()[esel], gres[0].cpu().numpy())
    assert np.array_equal(st_b["j_stop"][esel], gres[2]["j_stop"]) and np.array_equal(st_b["evaluated"][esel], gres[2]["evaluated"])
