"""Host-side checks of the C-ABI library (no GPU): it loads, exports every symbol include/pfg.h
declares, and its host-only logic (the budget -> L cost model, R-11) behaves."""
import ctypes as C
import os
import re

import pytest

import paper_1906_12211_b200 as pfg
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pfg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pfg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = pfg.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(pfg.EXPORTED) == syms
    assert lib.pfg_abi_version() == 1


def _c_sizes():
    """sizeof of the header's structs as a C compiler sees them"""
    import shutil
    import subprocess
    import tempfile
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        pytest.skip("no C compiler")
    src = ('#include "pfg.h"\n#include <stdio.h>\nint main(void){printf("%zu %zu %zu %zu", sizeof(pfg_build_opts), '
           'sizeof(pfg_search_opts), sizeof(pfg_query_stats), sizeof(pfg_index_info_t)); return 0;}\n')
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "s.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "s")
        subprocess.check_call([cc, "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        return [int(x) for x in subprocess.check_output([exe]).split()]


def test_abi_struct_sizes_match_header():
    # the binding's ctypes mirrors must have the C sizes (struct_size versioning)
    b, s, q, i = _c_sizes()
    assert C.sizeof(pfg.BuildOpts) == b
    assert C.sizeof(pfg.SearchOpts) == s
    assert pfg.STATS_DTYPE.itemsize == q
    assert C.sizeof(pfg.IndexInfo) == i


def test_cost_model_tensor():
    # tensor: L is rounded down to an even power of two (at most 256); K must be an
    # even number of whole functions
    assert pfg.derive_reps(1_000_000, 100, "fht_cp", 4 << 30, strategy="tensor", prefix_bits=32)[0] == 64
    assert pfg.derive_reps(1_000_000, 100, "simhash", 64 << 30, strategy="tensor")[0] == 256
    with pytest.raises(pfg.PfgError):
        pfg.derive_reps(1_000_000, 100, "fht_cp", 4 << 30, strategy="tensor")      # 3 functions of 8 bits
    with pytest.raises(pfg.PfgError):
        pfg.derive_reps(10_000, 32, "simhash", 0, strategy="tensor", reps=32)      # not an even power of two


def test_cost_model_configs():
    # L for BASELINE configs 2-5 at their budgets (GiB) under the R-11 cost model with 16-byte
    # entries (R-21); SURVEY.md Appendix B has the 8-byte-entry figures 452 / 884 / 1626 / 1206
    assert pfg.derive_reps(1_000_000, 100, "fht_cp", 4 << 30)[0] == 241  # 16-byte entries with inline sketch words (R-21)
    assert pfg.derive_reps(1_000_000, 300, "simhash", 8 << 30)[0] == 458
    assert pfg.derive_reps(1_000_000, 960, "simhash", 16 << 30, strategy="pool")[0] == 830
    assert pfg.derive_reps(12_500_000, 100, "fht_cp", 120 << 30)[0] == 618


def test_cost_model_arithmetic():
    # budget = fixed + exactly 3 repetitions -> L = 3; one byte less -> 2
    L, minb, ib = pfg.derive_reps(5000, 40, "simhash", 10 << 30, max_reps=1)
    per_rep = 16 * 5000 + 4 * 8193 + 1 + 24 * 4 * 40
    fixed = minb - per_rep
    assert pfg.derive_reps(5000, 40, "simhash", fixed + 3 * per_rep)[0] == 3
    assert pfg.derive_reps(5000, 40, "simhash", fixed + 3 * per_rep - 1)[0] == 2
    assert pfg.derive_reps(5000, 40, "simhash", 1 << 40)[0] == 4096  # cap
    assert pfg.derive_reps(5000, 40, "simhash", 1 << 40, max_reps=100)[0] == 100


def test_cost_model_budget_error_names_minimum():
    with pytest.raises(pfg.PfgError, match=r"minimum is \d+ B") as e:
        pfg.derive_reps(1_000_000, 100, "fht_cp", 100 << 20)
    assert e.value.status == 3


@pytest.mark.parametrize("kw,msg", [
    (dict(prefix_bits=40), "prefix_bits"), (dict(sketch_words=65), "sketch_words"),
    (dict(strategy=7), "strategy"), (dict(cp_draws=-5), "cp_draws")])
def test_bad_options_rejected(kw, msg):
    with pytest.raises(pfg.PfgError, match=msg):
        pfg.derive_reps(1000, 16, "simhash", 1 << 30, **kw)


def test_bad_shapes_rejected():
    with pytest.raises(pfg.PfgError, match="n must"):
        pfg.derive_reps(0, 16, "simhash", 1 << 30)
    with pytest.raises(pfg.PfgError, match="d must"):
        pfg.derive_reps(10, 0, "simhash", 1 << 30)
    with pytest.raises(pfg.PfgError, match="d <= 1024"):
        pfg.derive_reps(10, 2000, "fht_cp", 1 << 30)


def test_config_records_carry_the_cost_model_L():
    # synth.CONFIGS records the budget-derived L (R-11) so that the CPU oracle legs of
    # bench.py need not load the product library; the record must equal the library's cost model
    import synth
    for cfg, c in synth.CONFIGS.items():
        if c["reps"]:
            continue
        n = c.get("shard_n", c["n"])
        assert c["L"] == pfg.derive_reps(n, c["d"], c["family"], c["budget"], strategy=c["strategy"])[0], cfg
