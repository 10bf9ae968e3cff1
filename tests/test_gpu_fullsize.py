"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times:
config 1 completely, config 2 (1M x 100, FHT cross-polytope, 4 GiB budget -> L = 241) on sampled
outputs the oracle computes one by one -- three whole repetition tables, the normalised data, and
the complete searches of 200 queries (the oracle builds only the repetitions they touch)."""
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
    orr = o.search(q, c["k"], c["recall"], rep_chunk=8, trace_cap=cap)
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
    sel = np.arange(0, len(q), 50)
    sub = (ids[sel], sims[sel], st[sel], tr[sel])
    orr = o.search(q[sel], c["k"], c["recall"], rep_chunk=8, trace_cap=cap, threads=1)
    _search_equal(sub, orr, cap)
