"""The reference's own harness and types on the GPU path: strsort.bench.run
(bench.py:311-355) and strsort-bench's main (cli.py:36-69) with the
gpu-s5 / gpu-ps5 algorithms registered through the plugin API
(register_algorithm, bench.py:151-152), and reference StringSet objects
(strset.py:34-89) passed through the drop-in entry points.

strsort comes from baseline/_ref (the reference package installed offline
into the repo, git-ignored, shipped to the GPU box) -- /root/reference is
never read here.  Skipped when it is not installed."""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
if REF.is_dir() and str(REF) not in sys.path:
    sys.path.insert(0, str(REF))
strsort = pytest.importorskip("strsort")
import strsort.bench as B  # noqa: E402
import strsort.cli as CLI  # noqa: E402
from strsort.strset import StringSet as RefStringSet  # noqa: E402

import paper_1403_2056_b200 as P  # noqa: E402
from paper_1403_2056_b200.bench_api import register_with_strsort  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _registered():
    assert register_with_strsort()


@pytest.mark.parametrize("algo,threads", [("gpu-s5", 1), ("gpu-ps5", 4)])
def test_bench_run_verifies(algo, threads):
    """RunConfig(algorithm=..., generator="random", n=10**6, verify=True):
    the reference harness times the GPU sort and checks it with its own
    verify (strset.py:250-281)."""
    res = B.run(B.RunConfig(algorithm=algo, generator="random", n=10**6, verify=True,
                            threads=threads, reps=2, counters=True))
    assert res.verify_ok is True
    assert res.n == 10**6 and len(res.times) == 2
    assert res.D is not None and res.L is not None  # counters=True: dist_stats of the output


def test_bench_run_suffixes_verifies():
    res = B.run(B.RunConfig(algorithm="gpu-s5", generator="suffix", n=50_000, verify=True))
    assert res.verify_ok is True


def test_cli_with_gpu_algorithm(capsys):
    rc = CLI.main(["--algo", "gpu-s5", "--gen", "random", "--n", "200000", "--verify",
                   "--format", "csv"])
    assert rc == 0
    out = capsys.readouterr().out
    assert "gpu-s5" in out and "pass" in out


def test_reference_stringset_through_drop_in():
    """A reference StringSet in, reference-compatible results out -- equal to
    the reference's own s5_sort (imported from baseline/_ref) bit for bit."""
    from strsort.ssss import s5_sort as ref_s5_sort

    rng = np.random.default_rng(11)
    items = [bytes(rng.integers(97, 101, size=int(rng.integers(0, 12)), dtype=np.uint8))
             for _ in range(3000)]
    buf = b"".join(x + b"\0" for x in items)
    starts = np.concatenate(([0], np.cumsum([len(x) + 1 for x in items])[:-1])).astype(np.int64)
    rs = RefStringSet(buf, starts)
    want = ref_s5_sort(rs, want_lcps=True, want_dchar=True)
    got = P.s5_sort(rs, want_lcps=True, want_dchar=True)
    assert np.array_equal(got.set.handles, want.set.handles)
    assert np.array_equal(got.lcps, want.lcps) and np.array_equal(got.dchar, want.dchar)
    assert isinstance(got.set, RefStringSet) and got.set.buffer is rs.buffer
    plain = P.s5_sort(rs)
    assert isinstance(plain, RefStringSet) and np.array_equal(plain.handles, want.set.handles)
    par = P.parallel_s5(rs, p=1, want_lcps=True)
    assert np.array_equal(par.set.handles, want.set.handles) and np.array_equal(par.lcps, want.lcps)
