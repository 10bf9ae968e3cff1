"""Pins of the CPU oracle against what the paper and mathematics fix (not against itself).

Each test names the PAPER.md passage (or DESIGN.md reading R-n) and the kind of pin:
golden value, closed form, invariant, brute force, or an independent re-implementation in
numpy of a textbook definition (Sylvester Hadamard matrix, exact sorting, exact k-NN).
"""
import math

import numpy as np
import pytest

import oracle as O
import synth
from conftest import golden


def _rows(path):
    out = []
    for line in open(path):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line.split())
    return out


# ---------------------------------------------------------------- a1 normalise
def test_normalize_golden_and_zero_row():
    # SPEC.md:47 worked example, "We normalize ... all data vectors"
    out = O.normalize(np.array([[3.0, 4.0]], np.float32))
    assert out[0, 0] == np.float32(0.6) and out[0, 1] == np.float32(0.8)
    with pytest.raises(ZeroDivisionError, match="row 1"):
        O.normalize(np.array([[1.0, 0.0], [0.0, 0.0]], np.float32))


def test_normalize_unit_norm_and_idempotent():
    x = np.random.default_rng(0).standard_normal((500, 37)).astype(np.float32) * 7
    y = O.normalize(x)
    assert np.allclose(np.linalg.norm(y.astype(np.float64), axis=1), 1.0, atol=1e-6)
    z = O.normalize(y)
    assert np.max(np.abs(z.view(np.int32) - y.view(np.int32))) <= 1  # within 1 ulp


# ---------------------------------------------------------------- canonical dot (R-2)
def test_dot_close_to_double():
    rng = np.random.default_rng(1)
    a = O.normalize(rng.standard_normal((200, 100)))
    b = O.normalize(rng.standard_normal((200, 100)))
    for i in range(200):
        ref = float(np.dot(a[i].astype(np.float64), b[i].astype(np.float64)))
        assert abs(O.dot(a[i], b[i]) - ref) < 1e-6
        assert abs(O.sim(a[i], b[i]) - ref) < 1e-6
    assert O.dot(np.array([1, 2, 3], np.float32), np.array([4, 5, 6], np.float32)) == 32.0


def test_sim_exact_on_integers_and_long_vectors():
    # integer-valued products are exact in fp32, so any summation order gives the exact sum;
    # covers d > 128 (several chunks per lane) and d not a multiple of 4
    rng = np.random.default_rng(8)
    for d in (1, 3, 7, 100, 129, 300, 960, 1030):
        a = rng.integers(-8, 9, size=d).astype(np.float32)
        b = rng.integers(-8, 9, size=d).astype(np.float32)
        assert O.sim(a, b) == float(np.dot(a.astype(np.int64), b.astype(np.int64)))
    x = O.normalize(rng.standard_normal((50, 960)))
    for i in range(49):
        assert abs(O.sim(x[i], x[i + 1]) - float(x[i].astype(np.float64) @ x[i + 1].astype(np.float64))) < 2e-6
    assert abs(O.sim(x[0], x[0]) - 1.0) < 1e-6


# ---------------------------------------------------------------- HP
def test_hp_bit_definition():
    assert O.hp_bit([1, 0], [1, 0]) == 1 and O.hp_bit([1, 0], [-1, 0]) == 0
    assert O.hp_bit([1, 0], [0, 1]) == 1  # <a,x> = 0 counts as ">= 0" (R-4)


def test_hp_collision_closed_form():
    # Charikar: Pr[h(x) = h(y)] = 1 - theta/pi; the oracle's Monte-Carlo routine with the HP
    # family (1 bit) must reproduce it on the whole alpha grid
    T = O.cp_table(O.HP, 16, seed=5, draws=20000)
    for a in range(41):
        alpha = min(1.0, -1.0 + 0.05 * a)
        assert abs(T[1, a] - (1 - math.acos(alpha) / math.pi)) < 0.02, a


# ---------------------------------------------------------------- FHT (R-6)
def _sylvester(n):
    H = np.array([[1.0]])
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


@pytest.mark.parametrize("dp", [2, 8, 32, 128, 512])
def test_fht_is_sylvester_hadamard(dp):
    rng = np.random.default_rng(dp)
    x = rng.standard_normal(dp).astype(np.float32)
    y = O.fht(x)
    ref = _sylvester(dp) @ x.astype(np.float64)
    assert np.allclose(y, ref, rtol=0, atol=1e-4 * math.sqrt(dp))
    # involution up to scale: H H = dp I; Parseval |Hx|^2 = dp |x|^2
    assert np.allclose(O.fht(y), dp * x, atol=1e-3 * dp)
    assert abs(np.sum(y.astype(np.float64) ** 2) - dp * np.sum(x.astype(np.float64) ** 2)) < 1e-3 * dp * dp


def test_fhtcp_code_basis_vector_and_sign_msb():
    # all-+ signs, x = e_0: H H H e_0 = dp * (1,...,1) -> all |y_u| tie -> axis 0, positive
    dp = 128
    x = np.zeros(100, np.float32); x[0] = 1
    assert O.fhtcp_code(x, dp, np.ones(3 * dp, np.float32)) == 0
    # R-5: the sign is the MSB of ell = 1 + log2 dp = 8 bits; -x flips only that bit
    rng = np.random.default_rng(3)
    for _ in range(50):
        v = rng.standard_normal(100).astype(np.float32)
        s = np.where(rng.random(3 * dp) < .5, -1, 1).astype(np.float32)
        c1, c2 = O.fhtcp_code(v, dp, s), O.fhtcp_code(-v, dp, s)
        assert c1 ^ c2 == 0x80


def test_fhtcp_code_matches_explicit_rotation():
    # y = H D3 H D2 H D1 x with explicit matrices in double; code = argmax |y| + sign
    rng = np.random.default_rng(4)
    d, dp = 100, 128
    H = _sylvester(dp)
    for _ in range(100):
        v = rng.standard_normal(d).astype(np.float32)
        s = np.where(rng.random(3 * dp) < .5, -1.0, 1.0)
        y = np.concatenate([v.astype(np.float64), np.zeros(dp - d)])
        for r in range(3):
            y = H @ (s[r * dp:(r + 1) * dp] * y)
        a = int(np.argmax(np.abs(y)))
        srt = np.sort(np.abs(y))
        if srt[-1] - srt[-2] < 1e-3 * srt[-1]:
            continue  # near-tie: fp32 vs double may legitimately differ
        assert O.fhtcp_code(v, dp, s.astype(np.float32)) == ((int(y[a] < 0) << 7) | a)


# ---------------------------------------------------------------- CP table
@pytest.fixture(scope="module")
def cp100():
    return O.cp_table(O.FHTCP, 100, seed=1, draws=1000)


def test_cp_table_invariants(cp100):
    T = cp100
    assert T.shape == (9, 41)
    assert np.all(T[0] == 1.0)                       # empty prefix always collides
    assert np.all(T[:, 40] == 1.0)                   # alpha = 1: identical points
    assert np.all(T[1:, 0] == 0.0)                   # alpha = -1, sign in MSB (R-5): never collide
    assert np.all(np.diff(T, axis=1) >= 0)           # monotone in alpha (Def. 1)
    assert np.all(np.diff(T, axis=0) <= 0)           # monotone in prefix length b


def test_cp_table_reestimate(cp100):
    # a 10x-draw re-estimate with another seed agrees within 3 standard errors + the cleaning slack
    T2 = O.cp_table(O.FHTCP, 100, seed=77, draws=10000)
    for b in (1, 4, 8):
        for a in (10, 20, 30, 36, 38):
            p = T2[b, a]
            se = math.sqrt(max(p * (1 - p), 1e-4) / 1000)
            assert abs(cp100[b, a] - p) <= 3 * se + 0.01, (b, a)


# ---------------------------------------------------------------- filter threshold (R-15)
def test_tau_golden():
    for ip, eps, t in _rows(golden("tau.txt")):
        assert O.tau(float(ip), float(eps)) == int(t), (ip, eps)


def test_grid_bucket_rounds_down():
    # PAPER.md:352 "round the distance down": ip .97 -> bucket .95 (a = 39); exact grid -> itself
    assert O.grid_bucket(0.97) == 39
    assert O.grid_bucket(np.float32(-1.0 + 0.05 * 38)) == 38
    assert O.grid_bucket(-1.0) == 0 and O.grid_bucket(1.0) == 40
    assert O.grid_bucket(0.949999) == 38


# ---------------------------------------------------------------- stop rule
@pytest.fixture(scope="module")
def tiny_hp():
    data = synth.gaussian(300, 16, 9)
    return O.OracleIndex(data, O.HP, L=4, seed=3, M=2)


def test_stop_rule_golden(tiny_hp):
    for row in _rows(golden("stop_rule.txt")):
        if row[0] in ("pool", "tensor", "twolevel"):
            continue
        ip, i, delta, rule, js = float(row[0]), int(row[1]), float(row[2]), int(row[3]), int(row[4])
        assert not tiny_hp.should_stop(i, js - 1, ip, delta, rule), row
        assert tiny_hp.should_stop(i, js, ip, delta, rule), row


def test_pool_stop_rule_golden():
    row = [r for r in _rows(golden("stop_rule.txt")) if r[0] == "pool"][0]
    ip, i, delta, m, js = float(row[1]), int(row[2]), float(row[3]), int(row[4]), int(row[5])
    data = synth.gaussian(200, 8, 2)
    X = O.OracleIndex(data, O.HP, L=2, seed=1, M=1, strategy=O.POOL, pool_bits=m)
    assert X.m == m
    assert not X.should_stop(i, js - 1, ip, delta)
    assert X.should_stop(i, js, ip, delta)


def test_tensor_stop_rule_golden():
    data = synth.gaussian(300, 8, 2)
    X = O.OracleIndex(data, O.HP, L=256, seed=1, M=1, strategy=O.TENSOR, lazy=True)
    for row in [r for r in _rows(golden("stop_rule.txt")) if r[0] == "tensor"]:
        ip, i, delta, ms = float(row[1]), int(row[2]), float(row[3]), int(row[4])
        assert not X.should_stop(i, ms - 1, ip, delta), row
        assert X.should_stop(i, ms, ip, delta), row


def test_tensor_interleave():
    # P12 / PAPER.md:247-248, 855-857: trie (j1, j2) hashes with the K/2 functions of tuple j1 of
    # the first collection and tuple j2 of the second, interleaved (first collection first).  The
    # functions are regenerated here from the shared seeded stream (R-3), the bits computed one by
    # one, and the interleaved codes compared with the index's codes for every trie.
    d, L, K = 12, 16, 4
    S, h = 4, K // 2
    data = synth.gaussian(50, d, 9)
    q = synth.gaussian(20, d, 10)
    X = O.OracleIndex(data, O.HP, L=L, K=K, seed=7, M=1, strategy=O.TENSOR)
    codes, _ = X.hash(q)
    key = O.stream_key(7, 1)                      # HP functions: stream tag 1 (R-3)
    qn = O.normalize(q)

    def fvec(f):
        return np.array([O.gauss_d(key, f * d + t) for t in range(d)], np.float32)

    for j1 in range(S):
        for j2 in range(S):
            funcs = []
            for s in range(h):
                funcs += [(0 * S + j1) * h + s, (1 * S + j2) * h + s]
            for r in range(len(q)):
                code = 0
                for f in funcs:
                    code = (code << 1) | O.hp_bit(fvec(f), qn[r])
                assert code == codes[r, j1 * S + j2], (j1, j2, r)


def test_tensor_recall_over_seeds():
    # Alg. 2's guarantee (filter off): config 1 with L = 16 tries from 2 x 4
    # tuples, index seeds 1..30, mean recall >= target
    data, q = synth.config_data(1, n=3000, nq=40)
    bi, _ = O.bruteforce(O.normalize(data), O.normalize(q), 10)
    rec = []
    for seed in range(1, 31):
        X = O.OracleIndex(data, O.HP, L=16, seed=seed, strategy=O.TENSOR)
        ids, _, tr = X.search(q, 10, 0.9, threads=8, use_filter=False)
        rec.append(np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ids.tolist(), bi.tolist())]))
        assert np.all(tr[:, 1] <= 4)          # at most S = 4 shells per depth
    assert np.mean(rec) >= 0.9, np.mean(rec)


def test_failure_bound_monotone(tiny_hp):
    # BJ: the failure bound decreases as j grows and as the prefix shrinks (fixed j)
    for ip in (0.3, 0.6, 0.9):
        for delta in (0.5, 0.1, 0.01):
            js = {}
            for i in range(1, 25):
                hi = 1
                while not tiny_hp.should_stop(i, hi, ip, delta):
                    hi *= 2
                lo = hi // 2        # should_stop(lo) is False (or lo == 0)
                while hi - lo > 1:
                    mid = (lo + hi) // 2
                    lo, hi = (lo, mid) if tiny_hp.should_stop(i, mid, ip, delta) else (mid, hi)
                js[i] = hi
                # monotone in j: every later j also stops
                assert all(tiny_hp.should_stop(i, hi + s, ip, delta) for s in (1, 7, 1000))
            assert all(js[i] <= js[i + 1] for i in range(1, 24))
    P = [tiny_hp.P(i, 0.7) for i in range(25)]
    assert P[0] == 1.0 and all(P[i] > P[i + 1] for i in range(24))


# ---------------------------------------------------------------- widening
def test_widen_golden():
    codes = np.array([0, 1, 4, 6], np.uint32)
    state = {}
    for qc, i, lo, hi in _rows(golden("widen.txt")):
        qc, i, lo, hi = int(qc), int(i), int(lo), int(hi)
        if i == 3:
            p = O.lower_bound(codes, qc)
            state[qc] = (p, p)
        state[qc] = O.widen(codes, qc, 3, i, 1, *state[qc])
        assert state[qc] == (lo, hi), (qc, i)


def test_widen_properties():
    # superset of exact prefix matches, overshoot <= B-1 per side (<= 2(B-1) per step),
    # monotone, level 0 emits everything
    rng = np.random.default_rng(7)
    K = 10
    for B in (1, 3, 12):
        codes = np.sort(rng.integers(0, 1 << K, size=800)).astype(np.uint32)
        for qc in rng.integers(0, 1 << K, size=40):
            p = O.lower_bound(codes, int(qc))
            assert p == np.searchsorted(codes, qc, side="left")
            lo, hi = p, p
            for i in range(K, -1, -1):
                nlo, nhi = O.widen(codes, int(qc), K, i, B, lo, hi)
                assert nlo <= lo and nhi >= hi
                m = np.nonzero((codes >> (K - i)) == (int(qc) >> (K - i)))[0]
                if m.size:
                    assert nlo <= m[0] and nhi >= m[-1] + 1
                    assert m[0] - nlo <= B - 1 or nlo == lo
                    assert nhi - (m[-1] + 1) <= B - 1 or nhi == hi
                if B == 1 and m.size:
                    assert (nlo, nhi) == (m[0], m[-1] + 1)
                lo, hi = nlo, nhi
            assert (lo, hi) == (0, codes.size)


# ---------------------------------------------------------------- index structure
@pytest.fixture(scope="module")
def small_fht():
    data, q = synth.config_data(2, n=3000, nq=40)
    return O.OracleIndex(data, O.FHTCP, L=12, seed=5), data, q


def test_tables_sorted_permutation(small_fht):
    X, data, _ = small_fht
    codes_all, _ = X.hash(data)             # rep codes of every point, computed point by point
    for j in (0, 5, 11):
        c, ids = X.rep(j)
        order = np.lexsort((np.arange(X.n), codes_all[:, j]))   # numpy: sort by (code, id)
        assert np.array_equal(ids, order.astype(np.uint32))
        assert np.array_equal(c, codes_all[order, j])
        pt = X.prefix_table(j)
        ref = np.searchsorted(c >> 11, np.arange(8193), side="left")
        assert np.array_equal(pt, ref.astype(np.uint32))
    assert X.ell == 8 and X.c == 3 and X.dp == 128


def test_rep_code_sign_structure(small_fht):
    # FHT-CP rep code = 3 concatenated 8-bit codes with the sign at each MSB (R-5, R-7):
    # negating the input flips exactly bits 23, 15, 7
    X, data, _ = small_fht
    c1, _ = X.hash(data[:50])
    c2, _ = X.hash(-data[:50])
    assert np.all((c1 ^ c2) == 0x808080)


def test_sketch_properties():
    data = synth.gaussian(64, 40, 3)
    X = O.OracleIndex(data, O.HP, L=2, seed=1, M=32)
    _, s1 = X.hash(data)
    _, s2 = X.hash(-data)
    assert np.all(s1 == X.sketches())
    flips = np.vectorize(lambda v: bin(int(v)).count("1"))(s1 ^ s2)
    assert np.all(flips == 64)                             # v vs -v: every hyperplane separates
    rng = np.random.default_rng(0)
    a = rng.standard_normal(40); b = rng.standard_normal(40); b -= a * (a @ b) / (a @ a)
    _, sa = X.hash(a[None].astype(np.float32)); _, sb = X.hash(b[None].astype(np.float32))
    ham = np.vectorize(lambda v: bin(int(v)).count("1"))(sa ^ sb)
    assert abs(ham.mean() - 32) < 4                        # orthogonal: Binomial(64, 1/2)


# ---------------------------------------------------------------- brute force / search
def test_bruteforce_vs_numpy():
    rng = np.random.default_rng(2)
    x = O.normalize(rng.standard_normal((700, 24)))
    q = O.normalize(rng.standard_normal((30, 24)))
    ids, sims = O.bruteforce(x, q, 7)
    S = q.astype(np.float64) @ x.astype(np.float64).T
    for i in range(30):
        order = np.lexsort((np.arange(700), -S[i]))[:7]
        assert np.array_equal(ids[i], order)
        assert np.allclose(sims[i], S[i, order], atol=1e-12)


@pytest.mark.parametrize("family", [O.HP, O.FHTCP])
def test_exactness_at_exhaustion(family):
    # recall 1 -> delta = 0: the stop rule cannot fire above i = 0, whose linear scan (R-13,
    # PAPER.md:221) returns the exact k-NN, ties by id
    data, q = synth.config_data(1, n=1500, nq=25)
    X = O.OracleIndex(data, family, L=3, seed=2)
    ids, sims, tr = X.search(q, 10, 1.0, rep_chunk=2)
    bi, bs = O.bruteforce(X.data(), O.normalize(q), 10)
    assert np.array_equal(ids, bi)
    assert np.allclose(sims, bs, atol=1e-6)
    assert np.all(tr[:, 0] == 0) and np.all(tr[:, 5] == 1500)


def test_k_greater_than_n_pads():
    data, q = synth.config_data(1, n=5, nq=2)
    X = O.OracleIndex(data, O.HP, L=2, seed=2)
    ids, sims, tr = X.search(q, 8, 0.9)
    assert np.all(ids[:, 5:] == -1) and np.all(np.isneginf(sims[:, 5:]))
    assert set(ids[0, :5]) == set(range(5)) and np.all(tr[:, 6] & 1)


def test_filter_off_equals_infinite_eps():
    # eps = +inf (tau = 64) gives the same output as the filter off
    data, q = synth.config_data(1, n=2000, nq=20)
    X = O.OracleIndex(data, O.HP, L=8, seed=4)
    a = X.search(q, 10, 0.8, rep_chunk=3, use_filter=False)
    b = X.search(q, 10, 0.8, rep_chunk=3, eps=1e9, tau_rule=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2][:, :2], b[2][:, :2])


def test_chunk_schedule_only_moves_tau():
    # R-17: the chunk schedule (the single repetition 0, then chunks of R; or uniform chunks of R)
    # only decides when tau is refreshed.  With the filter off it
    # cannot change the search at all, and with R = 1 both schedules are the same chunks.
    data, q = synth.config_data(1, n=2000, nq=20)
    X = O.OracleIndex(data, O.HP, L=8, seed=4)
    ref = X.search(q, 10, 0.8, rep_chunk=1, use_filter=False)
    for R in (1, 3, 8):
        for uni in (False, True):
            r = X.search(q, 10, 0.8, rep_chunk=R, use_filter=False, uniform_chunks=uni)
            assert np.array_equal(r[0], ref[0]) and np.array_equal(r[2], ref[2]), (R, uni)
    a = X.search(q, 10, 0.8, rep_chunk=1)
    b = X.search(q, 10, 0.8, rep_chunk=1, uniform_chunks=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
    # with the filter, the default schedule sets tau after repetition 0 instead of after R, so the
    # filter rejects more
    d2, q2 = synth.config_data(2, n=4000, nq=30)
    X2 = O.OracleIndex(d2, O.FHTCP, L=16, seed=1)
    c = X2.search(q2, 10, 0.9, rep_chunk=8)
    u = X2.search(q2, 10, 0.9, rep_chunk=8, uniform_chunks=True)
    assert np.sum(c[2][:, 3]) > np.sum(u[2][:, 3])  # more rejections by the filter
    assert np.sum(c[2][:, 5]) < np.sum(u[2][:, 5])  # fewer exact evaluations


def test_trace_accounting_and_lemma1():
    data, q = synth.config_data(2, n=4000, nq=30)
    X = O.OracleIndex(data, O.FHTCP, L=16, seed=1)
    ids, sims, tr, tids = X.search(q, 10, 0.9, rep_chunk=4, trace_cap=4000)
    # emitted = filtered + dups + evaluated
    assert np.all(tr[:, 2] == tr[:, 3] + tr[:, 4] + tr[:, 5])
    bi, bs = O.bruteforce(X.data(), O.normalize(q), 10)
    for r in range(30):
        ev = tids[r, : tr[r, 5]]
        assert len(set(ev.tolist())) == tr[r, 5]
        # the returned list is exactly the top-10 of the evaluated set (Alg. 1 PQ)
        s = np.array([O.sim(O.normalize(q[r:r + 1])[0], X.data()[e]) for e in ev], np.float32)
        order = np.lexsort((ev, -s))[:10]
        assert np.array_equal(ids[r], ev[order].astype(np.int64))
        # Lemma 1 invariant: the found k-th similarity never exceeds the true k-th
        assert sims[r, 9] <= bs[r, 9] + 1e-6


def test_recall_over_100_seeds():
    # BJ / P11: config 1 (n=10K, d=32, SimHash, L=32, recall target .9), index seeds 1..100, with the
    # search options bench.py uses (R = 16, default chunk schedule, the sketch filter with the
    # default quantile threshold of R-26): mean recall >= .9.  Lemma 1
    # proves the guarantee for Alg. 1 without the filter, pinned as well.  The
    # expected-distance threshold of the paper's eps = 0 experiments (R-15) loses
    # recall (.08 to .03 in the paper) and is pinned only to the target minus .03.
    data, q = synth.config_data(1)
    qn = O.normalize(q)
    bi, _ = O.bruteforce(O.normalize(data), qn, 10)
    rec = {"off": [], "quantile": [], "expected": []}
    for seed in range(1, 101):
        X = O.OracleIndex(data, O.HP, L=32, seed=seed)
        for name, kw in (("off", dict(use_filter=False)), ("quantile", dict()), ("expected", dict(tau_rule=1))):
            ids, _, _ = X.search(q, 10, 0.9, rep_chunk=16, threads=8, **kw)
            rec[name].append(np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ids.tolist(), bi.tolist())]))
    assert np.mean(rec["off"]) >= 0.9, np.mean(rec["off"])
    assert np.mean(rec["quantile"]) >= 0.9, np.mean(rec["quantile"])
    assert np.mean(rec["expected"]) >= 0.9 - 0.03, np.mean(rec["expected"])


def test_planted_hit_rate():
    # SPEC.md:198 / P11: the planted partner (the true 1-NN) is found with probability
    # >= 1 - delta - .02 over index rebuilds (filter off: the proven Alg. 1 setting)
    data, q, rows = synth.planted(4000, 64, 40, seed=11, stride=100)
    bi, _ = O.bruteforce(O.normalize(data), O.normalize(q), 1)
    assert np.all(bi[:, 0] == rows)
    hits = trials = 0
    for seed in range(1, 21):
        X = O.OracleIndex(data, O.HP, L=16, seed=seed, M=8)
        ids, _, _ = X.search(q, 1, 0.9, threads=8, use_filter=False)
        hits += int(np.sum(ids[:, 0] == rows)); trials += len(rows)
    assert hits / trials >= 0.9 - 0.02, hits / trials


# ---------------------------------------------------------------- generators (P14)
def test_generator_planted():
    data, q, rows = synth.planted(20000, 300, 200, seed=3)
    qd = q.astype(np.float64)
    cos = np.sum(qd * data[rows].astype(np.float64), axis=1)
    assert np.allclose(cos, 0.6, atol=1e-6)
    S = qd @ data.astype(np.float64).T
    assert np.mean(np.argmax(S, axis=1) == rows) >= 0.999


def test_generator_paper_synthetic():
    # x_n is the nearest neighbour; E<q_i,x_n> = 1/2, E<q_i,x_j> = 0
    data, q = synth.paper_synthetic(5000, 100, 1000, seed=1)
    S = q.astype(np.float64) @ data.astype(np.float64).T
    assert abs(S[:, -1].mean() - 0.5) < 0.02
    assert abs(S[:, :-1].mean()) < 0.02
    assert np.mean(np.argmax(S, axis=1) == 4999) >= 0.99


# ------------------------------------------------------------------ R-25 16-bit fixed point
def test_fixed16_golden():
    # insert((1,0,0)) -> (32767, 0, 0) (round(1 * 2^15) clamped); -1 is representable;
    # ties go to even (rint under the default rounding mode)
    v = np.array([1.0, 0.0, -1.0, 0.5, -0.25, 1.5 / 32768, 2.5 / 32768, -0.5 / 32768, -1.5 / 32768, 0.999999],
                 np.float32)
    assert O.fixed16(v).tolist() == [32767, 0, -32768, 16384, -8192, 2, 2, 0, -2, 32767]


def test_sim16_within_spec_bound_of_double():
    # for 10^4 random unit-vector pairs |fixed - float inner product| <= 2e-3
    rng = np.random.default_rng(11)
    a = O.normalize(rng.standard_normal((10_000, 100)).astype(np.float32))
    b = O.normalize(rng.standard_normal((10_000, 100)).astype(np.float32))
    a16, b16 = O.fixed16(a.ravel()).reshape(a.shape), O.fixed16(b.ravel()).reshape(b.shape)
    err = max(abs(O.sim16(a16[i], b16[i]) - float(a[i].astype(np.float64) @ b[i].astype(np.float64)))
              for i in range(0, 10_000, 7))
    assert err <= 2e-3
    # exact integer arithmetic: symmetric, and a unit vector with itself within the rounding of d
    # coordinates (|q - x 2^15| <= 1/2 each)
    assert O.sim16(a16[0], b16[0]) == O.sim16(b16[0], a16[0])
    assert abs(O.sim16(a16[3], a16[3]) - 1.0) <= 100 * 2.0 ** -15


def test_sim16_is_the_exact_integer_sum():
    # the scaled sum equals the int64 dot of the codes (numpy) rounded to fp32 -- no summation
    # order enters (R-25)
    rng = np.random.default_rng(5)
    a = O.fixed16(O.normalize(rng.standard_normal((1, 960)).astype(np.float32)).ravel())
    b = O.fixed16(O.normalize(rng.standard_normal((1, 960)).astype(np.float32)).ravel())
    exact = int(np.dot(a.astype(np.int64), b.astype(np.int64)))
    assert O.sim16(a, b) == np.float32(exact) * np.float32(2.0 ** -30)


def test_int16_storage_recall_on_config1():
    # the adaptive search with fixed-point inner products still meets the recall target (filter on)
    c = synth.CONFIGS[1]
    data, q = synth.config_data(1)
    o = O.OracleIndex(data, O.HP, L=c["reps"], seed=1, storage="i16")
    ids, sims, tr = o.search(q, c["k"], c["recall"], rep_chunk=8, rerank=False)
    bi, bs = O.bruteforce(o.data(), O.normalize(q), c["k"])
    hit = np.mean([len(set(ids[r]) & set(bi[r])) / c["k"] for r in range(len(q))])
    assert hit >= 0.87
    # without the fp32 re-rank every returned similarity is the fixed-point inner product of that pair
    x16, q16 = o.data16(), O.fixed16(O.normalize(q).ravel()).reshape(q.shape)
    for r in range(0, len(q), 9):
        for t in range(c["k"]):
            assert sims[r, t] == np.float32(O.sim16(q16[r], x16[ids[r, t]]))


# ------------------------------------------------------------------ exact cross-polytope (NEXT-2)
def test_cp_code_identity_rotation():
    # with the identity as hyperplanes, the code is the index of the largest |coordinate| plus the
    # sign in the most significant bit (d = 8: ell = 4); ties go to the lowest index
    d, ell = 8, 4
    A = np.eye(d, dtype=np.float32)
    e = np.zeros(d, np.float32)
    e[3] = 1.0
    assert O.cp_code(A, e) == 3
    assert O.cp_code(A, -e) == (1 << (ell - 1)) | 3
    t = np.zeros(d, np.float32)
    t[1] = t[5] = -0.5
    assert O.cp_code(A, t) == (1 << (ell - 1)) | 1
    # a permutation of the hyperplanes permutes the index
    P = np.eye(d, dtype=np.float32)[[2, 0, 1, 3, 4, 5, 6, 7]]
    assert O.cp_code(P, e) == 3 and O.cp_code(P, np.eye(d, dtype=np.float32)[2]) == 0


def test_cp_exact_table_canonical_pair_vs_random_pairs():
    # the table uses the paper's canonical pair (spherical symmetry); a direct Monte
    # Carlo with full random hyperplane matrices and random pairs at the same alpha must agree
    d, draws = 16, 3000
    T = O.cp_table(O.CP, d, 3, draws)
    ell = T.shape[0] - 1
    assert ell == 1 + 4
    assert np.all(T[:, 40] == 1.0) and np.all(T[1:, 0] == 0.0)      # alpha = 1 and alpha = -1
    assert np.all(np.diff(T, axis=1) >= 0) and np.all(np.diff(T, axis=0) <= 0)
    rng = np.random.default_rng(7)
    for a in (24, 32):                                                # alpha = 0.2, 0.6
        alpha = -1.0 + 0.05 * a
        hits = 0
        n = 1500
        for _ in range(n):
            A = rng.standard_normal((d, d)).astype(np.float32)
            x = rng.standard_normal(d)
            x /= np.linalg.norm(x)
            u = rng.standard_normal(d)
            u -= (u @ x) * x
            u /= np.linalg.norm(u)
            y = alpha * x + np.sqrt(1 - alpha * alpha) * u
            hits += O.cp_code(A, x.astype(np.float32)) == O.cp_code(A, y.astype(np.float32))
        p = hits / n
        sd = np.sqrt(p * (1 - p) / n + T[ell, a] * (1 - T[ell, a]) / draws)
        assert abs(p - T[ell, a]) <= 4 * sd + 1e-3, (a, p, T[ell, a])


def test_cp_exact_index_recall():
    data, q = synth.config_data(1, n=2000, nq=40)
    data, q = data[:, :16].copy(), q[:, :16].copy()
    for strat in (O.INDEPENDENT, O.POOL):
        o = O.OracleIndex(data, O.CP, L=12, seed=2, strategy=strat, pool_bits=120, cp_draws=300)
        ids, sims, tr = o.search(q, 10, 0.9, rep_chunk=4)
        bi, _ = O.bruteforce(o.data(), O.normalize(q), 10)
        hit = np.mean([len(set(ids[r]) & set(bi[r])) / 10 for r in range(len(q))])
        assert hit >= 0.85, (strat, hit)


# ------------------------------------------------------------------ round 2 pins
def _fhtcp_codes_numpy(X, S, H, ell):
    """FHT-CP codes of the rows of X (float64, zero-padded to dp) under sign sets S [N, 3, dp]:
    y = H D3 H D2 H D1 x with the explicit Sylvester matrix, code = argmax |y|
    (lowest index on ties) with the sign as the most significant of ell bits (R-5)"""
    y = X
    for r in range(3):
        y = (S[:, r, :] * y) @ H
    a = np.argmax(np.abs(y), axis=1)
    neg = y[np.arange(len(a)), a] < 0
    return (neg.astype(np.int64) << (ell - 1)) | a


def _pairs(rng, N, d, dp, alpha):
    """N random pairs of unit vectors in the first d of dp coordinates with inner product alpha"""
    x = rng.standard_normal((N, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    u = rng.standard_normal((N, d))
    u -= np.sum(u * x, axis=1, keepdims=True) * x
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    y = alpha * x + math.sqrt(1 - alpha * alpha) * u
    pad = np.zeros((N, dp - d))
    return np.hstack([x, pad]), np.hstack([y, pad])


@pytest.mark.parametrize("alpha_cell", [32, 38])          # alpha = 0.6, 0.9 (grid cells)
def test_fhtcp_prefix_probability_composition(alpha_cell):
    # The oracle's FHT-CP collision probability of an i-bit prefix of a repetition code,
    # P_i = T_ell^floor(i/ell) * T_(i mod ell) (a prefix of i bits is floor(i/ell)
    # whole functions plus the top i mod ell bits of the next; independent functions multiply), is
    # compared with a direct Monte Carlo of i-bit prefix collisions of whole 24-bit repetition codes
    # (3 functions concatenated MSB first, R-7) -- prefixes that stop inside the first, second and
    # third function -- on random pairs at that inner product, with independent numpy draws.
    d, dp, ell, N = 100, 128, 8, 20000
    alpha = -1.0 + 0.05 * alpha_cell
    rng = np.random.default_rng(1000 + alpha_cell)
    H = _sylvester(dp)
    x, y = _pairs(rng, N, d, dp, alpha)
    cx = np.zeros(N, np.int64)
    cy = np.zeros(N, np.int64)
    for f in range(3):
        S = np.where(rng.random((N, 3, dp)) < 0.5, -1.0, 1.0)
        cx = (cx << ell) | _fhtcp_codes_numpy(x, S, H, ell)
        cy = (cy << ell) | _fhtcp_codes_numpy(y, S, H, ell)
    X = O.OracleIndex(synth.gaussian(64, d, 3), O.FHTCP, L=1, seed=5, M=1, cp_draws=20000, lazy=True)
    ip = float(np.float32(alpha) + np.float32(1e-6))      # inside the cell (rounded down to it)
    assert O.grid_bucket(ip) == alpha_cell
    T = X.cp()
    for i in (4, 12, 20):
        p_mc = float(np.mean((cx >> (24 - i)) == (cy >> (24 - i))))
        P = X.P(i, ip)
        # standard error of the table estimate (20 000 draws per cell), propagated through the product
        m, rbits = i // ell, i % ell
        te, tr = T[ell, alpha_cell], T[rbits, alpha_cell]
        rel = math.sqrt((m * m) * (1 - te) / (te * 20000) + ((1 - tr) / (tr * 20000) if rbits else 0.0))
        se = math.sqrt(p_mc * (1 - p_mc) / N + (P * rel) ** 2)
        assert abs(p_mc - P) <= 3 * se + 1e-4, (i, p_mc, P, se)


def test_cp_table_random_pairs_below_canonical_pair():
    # P5 / SURVEY Appendix A, R-14: FHT-CP is not rotation invariant; the paper's canonical pair
    # x = e_1, y = (alpha, sqrt(1 - alpha^2), 0, ...) overestimates the 8-bit
    # collision rate at alpha >= .9, and the oracle's table (random pairs in the first d
    # coordinates) must not.  Canonical rate by an independent numpy Monte Carlo.
    d, dp, ell, N = 100, 128, 8, 20000
    T = O.cp_table(O.FHTCP, d, seed=11, draws=20000)
    H = _sylvester(dp)
    rng = np.random.default_rng(77)
    for cell in (38, 39):                                  # alpha = .90, .95
        alpha = -1.0 + 0.05 * cell
        x = np.zeros((N, dp)); x[:, 0] = 1.0
        y = np.zeros((N, dp)); y[:, 0] = alpha; y[:, 1] = math.sqrt(1 - alpha * alpha)
        S = np.where(rng.random((N, 3, dp)) < 0.5, -1.0, 1.0)
        canon = float(np.mean(_fhtcp_codes_numpy(x, S, H, ell) == _fhtcp_codes_numpy(y, S, H, ell)))
        se = math.sqrt(canon * (1 - canon) / N + T[ell, cell] * (1 - T[ell, cell]) / 20000)
        assert T[ell, cell] < canon + 1 * se, (cell, T[ell, cell], canon)   # Appendix A: ~7 SE below at .95


def test_pool_selections_distinct_and_uniform():
    # P12 / PAPER.md:886 ("random subsets of size K from the pool"): each repetition's c functions
    # are distinct indices of the pool, and the selection is a uniform sample without replacement:
    # every ordered pair (first, second) of the m (m - 1) pairs equally likely (chi-square), every
    # index equally likely at every position
    from scipy.stats import chisquare
    m, K, L = 8, 3, 24000                                  # HP: 8 pool functions, 3 per repetition
    X = O.OracleIndex(synth.gaussian(20, 6, 1), O.HP, L=L, K=K, seed=9, M=1, strategy=O.POOL, pool_bits=m, lazy=True)
    sel = X.pool_sel()
    assert sel.shape == (L, K) and sel.min() >= 0 and sel.max() < m
    assert all(len(set(r)) == K for r in sel.tolist())
    for t in range(K):
        assert chisquare(np.bincount(sel[:, t], minlength=m)).pvalue > 1e-3, t
    pair = sel[:, 0] * m + sel[:, 1]
    cnt = np.bincount(pair, minlength=m * m).reshape(m, m)
    assert np.all(np.diag(cnt) == 0)
    assert chisquare(cnt[~np.eye(m, dtype=bool)]).pvalue > 1e-3


def test_pool_recall_close_to_independent():
    # P12 / SPEC.md:569: pooled functions (Alg. 3, m = 3072 bits) reach a recall within .05 of
    # independent functions at the same (K, L) (filter off, the proven setting), config 1 shape
    data, q = synth.config_data(1, n=5000, nq=60)
    bi, _ = O.bruteforce(O.normalize(data), O.normalize(q), 10)
    rec = {O.INDEPENDENT: [], O.POOL: []}
    for seed in range(1, 16):
        for strat in rec:
            X = O.OracleIndex(data, O.HP, L=32, seed=seed, strategy=strat, pool_bits=3072, M=1)
            ids, _, _ = X.search(q, 10, 0.9, rep_chunk=8, threads=8, use_filter=False)
            rec[strat].append(np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ids.tolist(), bi.tolist())]))
    ri, rp = np.mean(rec[O.INDEPENDENT]), np.mean(rec[O.POOL])
    assert ri >= 0.9 and abs(rp - ri) <= 0.05, (ri, rp)


def test_tau_prob_is_the_binomial_quantile():
    # R-26: tau = the smallest t with P[Binomial(64, acos(ip)/pi) <= t] >= 1 - delta,
    # i.e. the (1 - delta)-quantile of the sketch Hamming distance of a pair at the k-th similarity
    # (64 independent HP bits, each differing w.p. acos(ip)/pi) -- scipy's ppf
    from scipy.stats import binom
    for delta in (0.5, 0.1, 0.01):
        for ip in np.linspace(-0.99, 0.999, 57):
            p = math.acos(float(np.float32(ip))) / math.pi
            want = int(binom.ppf(1 - delta, 64, p))
            got = O.tau_prob(float(np.float32(ip)), delta)
            if got != want:   # only at an exact CDF boundary (within the 1e-12 slack) may they differ
                assert abs(binom.cdf(got, 64, p) - (1 - delta)) < 1e-9, (delta, ip, got, want)
    for row in _rows(golden("tau_prob.txt")):
        assert O.tau_prob(float(row[0]), float(row[1])) == int(row[2]), row
    # the median (delta = .5) is within one of the expected-distance rule of R-15 (eps = 0)
    for ip in np.linspace(-0.9, 0.99, 40):
        assert abs(O.tau_prob(float(ip), 0.5) - O.tau(float(ip))) <= 1


def test_sim_seq_is_the_sequential_chain():
    # O-11: plain order = one fmaf chain in ascending t (or_dot), within 1e-6 of the double dot;
    # the R-2 lane-tree order differs from it by rounding only
    rng = np.random.default_rng(5)
    for d in (1, 7, 32, 100, 300, 960):
        for _ in range(20):
            a = rng.standard_normal(d).astype(np.float32); a /= np.linalg.norm(a)
            b = rng.standard_normal(d).astype(np.float32); b /= np.linalg.norm(b)
            s = np.float32(0)
            for t in range(d):
                s = np.float32(np.float64(a[t]) * np.float64(b[t]) + np.float64(s))   # fmaf: one rounding
            assert O.sim_seq(a, b) == s
            assert abs(O.sim_seq(a, b) - O.sim(a, b)) <= 2e-6


def test_search_results_do_not_hinge_on_the_summation_order():
    # R-2 vs O-11: the oracle's search with plain-order similarities returns the same ids and stop
    # points as with the lane-tree order, except where similarities tie within 1e-6
    data, q = synth.config_data(1)
    X = O.OracleIndex(data, O.HP, L=32, seed=1)
    a_ids, a_s, a_tr = X.search(q, 10, 0.9, rep_chunk=16, threads=8)
    b_ids, b_s, b_tr = X.search(q, 10, 0.9, rep_chunk=16, threads=8, sim_order=1)
    xn, qn = X.data(), O.normalize(q)
    exc = 0
    for r in range(len(q)):
        if np.array_equal(a_ids[r], b_ids[r]) and np.array_equal(a_tr[r, :2], b_tr[r, :2]):
            assert np.all(np.abs(a_s[r] - b_s[r]) <= 2e-6)
            continue
        exc += 1
        # an exception must come from a near tie: the two lists' exact similarities agree rank by rank
        ea = np.sort(xn[a_ids[r]].astype(np.float64) @ qn[r].astype(np.float64))[::-1]
        eb = np.sort(xn[b_ids[r]].astype(np.float64) @ qn[r].astype(np.float64))[::-1]
        assert np.all(np.abs(ea - eb) <= 1e-6), r
    assert exc <= 2, exc


def test_two_level_stop_bound_golden_and_monotone():
    # SURVEY 8(f)4 / PAPER.md:218-221: the two-level bound (stop_rule 2) against hand-derived j*, no
    # later than the one-level bound, and never weaker after descending a level: stopping after all
    # L repetitions at depth i + 1 implies stopping after the first repetition at depth i
    data = synth.gaussian(300, 16, 9)
    X = O.OracleIndex(data, O.HP, L=32, seed=3, M=2, lazy=True)
    for row in [r for r in _rows(golden("stop_rule.txt")) if r[0] == "twolevel"]:
        ip, i, delta, L, js = float(row[1]), int(row[2]), float(row[3]), int(row[4]), int(row[5])
        assert X.L == L
        if js > 1:
            assert not X.should_stop(i, js - 1, ip, delta, 2), row
        assert X.should_stop(i, js, ip, delta, 2), row
    for ip in (0.3, 0.6, 0.8, 0.95):
        for delta in (0.5, 0.1, 0.01):
            for i in range(1, 24):
                for j in (1, 5, 17, 32):
                    if X.should_stop(i, j, ip, delta, 0):
                        assert X.should_stop(i, j, ip, delta, 2), (ip, delta, i, j)
                if X.should_stop(i + 1, 32, ip, delta, 2):
                    assert X.should_stop(i, 1, ip, delta, 2), (ip, delta, i)


def test_int16_rerank_scores_in_fp32():
    # SURVEY 8(f)3 / PAPER.md:300-304: with 16-bit rows the returned top-k is re-scored with the fp32
    # similarity (R-2 order) and re-sorted; the id set is the fixed-point search's
    data, q = synth.config_data(1, n=4000, nq=30)
    X = O.OracleIndex(data, O.HP, L=16, seed=2, storage="i16")
    a_ids, a_s, _ = X.search(q, 10, 0.9, rep_chunk=8, rerank=False)
    b_ids, b_s, _ = X.search(q, 10, 0.9, rep_chunk=8, rerank=True)
    xn, qn = X.data(), O.normalize(q)
    for r in range(len(q)):
        assert set(a_ids[r].tolist()) == set(b_ids[r].tolist())
        want = [O.sim(qn[r], xn[i]) for i in b_ids[r]]
        assert np.array_equal(b_s[r], np.array(want, np.float32))
        keys = [(-s, i) for s, i in zip(b_s[r].tolist(), b_ids[r].tolist())]
        assert keys == sorted(keys)


def test_fhtcp_recall_over_seeds_config2_shape():
    # Lemma 1 with the FHT cross-polytope family: the
    # stop rule's collision probabilities P_i come from the FHT-CP branch of or_P (Monte-Carlo table,
    # prefix composition T_ell^floor(i/ell) T_(i mod ell), R-14), so a mistake there (too large P_i:
    # early stops) shows as recall below the target.  Config 2's shape (100-d Gaussian mixture),
    # 10 000 points, L = 32, recall target .9, index seeds 1..30: mean recall >= .9 with the filter off
    # (the proven setting) and with the default quantile filter (R-26).
    data, q = synth.config_data(2, n=10000, nq=60)
    bi, _ = O.bruteforce(O.normalize(data), O.normalize(q), 10)
    rec = {"off": [], "quantile": []}
    for seed in range(1, 31):
        X = O.OracleIndex(data, O.FHTCP, L=32, seed=seed, lazy=True, cp_draws=1000)
        for name, kw in (("off", dict(use_filter=False)), ("quantile", dict())):
            ids, _, _ = X.search(q, 10, 0.9, rep_chunk=16, threads=8, **kw)
            rec[name].append(np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ids.tolist(), bi.tolist())]))
    assert np.mean(rec["off"]) >= 0.9, np.mean(rec["off"])
    assert np.mean(rec["quantile"]) >= 0.9, np.mean(rec["quantile"])
