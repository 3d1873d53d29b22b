"""C-ABI contract checks that need no GPU (-m "not gpu"): the in-tree library loads and
exports every function include/sinkhorn_b200.h declares; the host-only entry
sk_shard_rows follows the fixed block partition."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "sinkhorn_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:sk_status|void|const char|int32_t)\s*\**\s*(\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2206_07630_b200 import _lib, build
    build.build()
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2206_07630_b200 import _lib
    decl = header_functions()
    assert len(decl) >= 20, decl
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = [s for s in decl if s not in syms]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == decl


def test_status_strings_and_version(lib):
    assert lib.sk_version() == 1
    assert lib.sk_status_string(0) == b"SK_OK"
    assert lib.sk_status_string(6) == b"SK_EUNSUPPORTED"


def test_shard_rows_partition():
    from paper_2206_07630_b200 import shard_rows
    for n in (1, 7, 256, 1000, 262144, 262145):
        for W in (1, 2, 4, 8):
            spans = [shard_rows(n, r, W) for r in range(W)]
            assert spans[0][0] == 0
            for (r0, nl), (r1, _) in zip(spans, spans[1:]):
                assert r0 + nl == r1               # contiguous
            assert spans[-1][0] + spans[-1][1] == n  # covering
            # boundaries are shared by all world sizes (bit-identity across W)
            b8 = {r0 for r0, _ in (shard_rows(n, r, 8) for r in range(8))}
            assert {r0 for r0, _ in spans} <= b8 | {n}


def test_no_product_import_of_oracle():
    """The product path never imports, links or executes the oracle (tests/bench/smoke only)."""
    pkg = os.path.join(ROOT, "paper_2206_07630_b200")
    for dp, _, fs in os.walk(pkg):
        for fn in fs:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, fn), errors="ignore").read()
                for bad in ("import oracle", "from oracle", "sk_oracle", "libsk_oracle"):
                    assert bad not in txt, (fn, bad)


def test_reports_view_of_the_batched_host_reports():
    """sinkhorn_solve's batched reports: the structured-array view (Reports) gives the same
    per-problem dicts as the ctypes structs and whole columns as numpy arrays."""
    from paper_2206_07630_b200 import Reports, SkReport
    raw = (SkReport * 4)()
    for k in range(4):
        raw[k].iterations, raw[k].converged, raw[k].marginal_error = 10 + k, k % 2, 0.25 * k
        raw[k].dual_objective, raw[k].solve_ms = -1.5 * k, 2.0
    rep = Reports(raw)
    assert len(rep) == 4 and [r["iterations"] for r in rep] == [10, 11, 12, 13]
    assert rep[2] == raw[2].as_dict()
    assert rep.column("converged").tolist() == [0, 1, 0, 1]
    assert rep[1:3] == [raw[1].as_dict(), raw[2].as_dict()]
