# tcgen05 SimHash bits vs the oracle: query sketches and codes bit-exact on several shapes
import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, oracle as O, paper_1906_12211_b200 as pfg, synth, time
dev = torch.device("cuda:0")
for cfg, n, nq, fam, L in ((1, 3000, 300, "simhash", 16), (2, 20000, 500, "fht_cp", 24), (4, 3000, 200, "simhash", 8)):
    d, q = synth.config_data(cfg, n=n, nq=nq)
    g = pfg.Index(torch.from_numpy(d).to(dev), 0, fam, seed=3, reps=L)
    o = O.OracleIndex(d, O.HP if fam == "simhash" else O.FHTCP, L=L, seed=3)
    gc, gs = g.hash_queries(q)
    oc, os_ = o.hash(q)
    print(cfg, "codes equal", np.array_equal(gc, oc), "sketches equal", np.array_equal(gs, os_),
          "bad sketch words", int(np.sum(gs != os_)), flush=True)
    tab = g.export_table(0); codes, ids = o.rep(0)
    print(cfg, "table 0 equal", np.array_equal((tab[:, 0] >> np.uint64(32)).astype(np.uint32), codes),
          "inline sketch equal", np.array_equal(tab[:, 1], o.sketches()[ids, o.slots()[0]]), flush=True)
# timing of the query sketch GEMM alone (config 2 shape): via hash_queries_reps(1 rep)
d, q = synth.config_data(2, n=100000, nq=10000)
g = pfg.Index(torch.from_numpy(d).to(dev), 0, "fht_cp", seed=1, reps=8)
Q = torch.from_numpy(q).to(dev)
for _ in range(3): g.hash_queries_reps(Q, 1)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(20): g.hash_queries_reps(Q, 1)
torch.cuda.synchronize(); print("hash_queries_reps(1) ms", (time.perf_counter() - t) / 20 * 1e3)
