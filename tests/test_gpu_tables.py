"""GPU: whole cutoff tables and files against the reference's own table files.

``tests/golden/table_*.csv`` were written by the reference (``build_table`` + ``write_table``,
and ``zipfks tables`` for the full finite grid; ``tests/golden/make_tables.py``).  The engine's
table for the same arguments must give the same file: identical metadata, header and grid
rows, cutoffs within the tier-2 tolerance (1e-10 relative: every KS value agrees with the
reference's to ~1e-14, so a selected order statistic can differ from the reference's in its last
digits, which ``repr`` shows).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
RTOL = 1e-10

# same arguments as tests/golden/make_tables.py
TABLES = {
    "table_k20_s5.csv": dict(ns=(20, 50), gammas=(1.0, 1.5), k=20, base_seed=5, replicates=200, repetitions=1),
    "table_inf_s3.csv": dict(ns=(10, 100, 300), gammas=(1.5, 2.5), k=None, base_seed=3, replicates=300,
                             repetitions=2),
    "table_k1000_s8.csv": dict(ns=(40, 200), gammas=(0.5, 1.25), k=1000, base_seed=8, replicates=256,
                               repetitions=1),
}


@pytest.fixture(scope="module")
def zk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1305_6738_b200 as zk

    return zk


def assert_same_file(got: str, want: str) -> int:
    """Lines equal except cutoff columns, which agree within RTOL; returns the bit-equal count."""
    g_lines, w_lines = got.splitlines(), want.splitlines()
    assert len(g_lines) == len(w_lines)
    assert g_lines[:4] == w_lines[:4]
    exact = 0
    for g, w in zip(g_lines[4:], w_lines[4:]):
        gf, wf = g.split(","), w.split(",")
        assert gf[:3] == wf[:3]
        for a, b in zip(map(float, gf[3:]), map(float, wf[3:])):
            assert abs(a - b) <= RTOL * abs(b), (g, w)
            exact += a == b
    return exact


@pytest.mark.parametrize("name", sorted(TABLES))
def test_table_file_matches_reference(zk, name, tmp_path):
    kw = dict(TABLES[name])
    k = kw.pop("k")
    support = zk.Support.unbounded() if k is None else zk.Support.finite(k)
    table = zk.build_table(support=support, **kw)
    path = tmp_path / name
    zk.write_table(table, path)
    with open(os.path.join(GOLDEN, name), encoding="utf-8") as fh:
        want = fh.read()
    assert_same_file(path.read_text(encoding="utf-8"), want)
    loaded = zk.load_table(path)
    assert loaded.cells == table.cells and loaded.gammas == table.gammas and loaded.ns == table.ns


def test_cli_tables_full_finite_grid_matches_reference(tmp_path):
    out = tmp_path / "grid.csv"
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    res = subprocess.run([sys.executable, "-m", "paper_1305_6738_b200", "tables", "--k", "20", "--replicates",
                          "100", "--reps", "1", "--seed", "13", "--out", str(out), "--workers", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr
    assert res.stdout.count("cell gamma=") == 180
    assert "wrote" in res.stdout and "180 cells" in res.stdout
    with open(os.path.join(GOLDEN, "tables_k20_r100_s13.csv"), encoding="utf-8") as fh:
        want = fh.read()
    assert_same_file(out.read_text(encoding="utf-8"), want)
