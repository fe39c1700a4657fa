"""Cutoff-table CSV files (host only): byte format against the reference's own files.

The fixtures ``tests/golden/table_*.csv`` were written by the reference's ``write_table``
(``tests/golden/make_tables.py``); the format checks follow ``tests/test_tablefile.py`` of the
reference.
"""
import os

import pytest

import paper_1305_6738_b200 as zk
from paper_1305_6738_b200 import cli
from paper_1305_6738_b200.tablefile import TableFormatError, format_table, load_table, write_table

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = ["table_k20_s5.csv", "table_inf_s3.csv", "table_k1000_s8.csv", "tables_k20_r100_s13.csv"]

HEADER = "k_support,gamma,n,q90,q95,q99,q999"


def _read(name):
    with open(os.path.join(GOLDEN, name), encoding="utf-8") as fh:
        return fh.read()


@pytest.mark.parametrize("name", FIXTURES)
def test_reference_files_round_trip_byte_for_byte(name, tmp_path):
    table = load_table(os.path.join(GOLDEN, name))
    out = tmp_path / name
    write_table(table, out)
    assert out.read_text(encoding="utf-8") == _read(name)
    assert load_table(out) == table


def test_reference_grid_file_shape():
    table = load_table(os.path.join(GOLDEN, "tables_k20_r100_s13.csv"))
    assert table.support == zk.Support.finite(20)
    assert table.gammas == cli.REFERENCE_GAMMAS_FINITE
    assert table.ns == cli.REFERENCE_NS
    assert len(table.cells) == 180
    assert (table.replicates, table.repetitions, table.base_seed) == (100, 1, 13)


def test_unbounded_label_and_lookup(tmp_path):
    table = zk.CutoffTable(support=zk.Support.unbounded(), levels=zk.DEFAULT_LEVELS, gammas=(1.25,), ns=(10,),
                           cells={(1.25, 10): (0.2792, 0.3092, 0.3668, 0.4315)}, replicates=50000,
                           repetitions=10, base_seed=1)
    path = tmp_path / "inf.csv"
    write_table(table, path)
    assert path.read_text().splitlines() == ["# replicates=50000", "# repetitions=10", "# seed=1", HEADER,
                                             "inf,1.25,10,0.2792,0.3092,0.3668,0.4315"]
    loaded = load_table(path)
    assert loaded == table and loaded.support.k is None
    assert loaded.cutoff(1.25, 10, 0.9) == 0.2792


def test_non_default_levels_rejected(tmp_path):
    table = zk.CutoffTable(support=zk.Support.finite(5), levels=(0.9, 0.95), gammas=(1.0,), ns=(10,),
                           cells={(1.0, 10): (0.1, 0.2)})
    with pytest.raises(TableFormatError, match="schema holds levels"):
        format_table(table)


@pytest.mark.parametrize("text, match", [
    ("# seed=1\nk_support,gamma,n,q90,q95,q99\n20,1.0,10,0.1,0.2,0.3\n", "header"),
    (HEADER + "\n20,1.0,10,0.2,0.1,0.3,0.4\n", "nondecreasing"),
    (HEADER + "\n20,1.0,10,0.1,0.2,0.3\n", "7 columns"),
    (HEADER + "\n20,1.0,10,0.1,0.2,0.3,0.4\n50,1.0,10,0.1,0.2,0.3,0.4\n", "mixed"),
    (HEADER + "\n20,1.0,10,0.1,0.2,0.3,0.4\n20,1.5,20,0.1,0.2,0.3,0.4\n", "incomplete"),
    (HEADER + "\n20,1.0,10,0.1,0.2,0.3,0.4\n20,1.0,10,0.1,0.2,0.3,0.4\n", "duplicate"),
    ("", "missing header"),
    (HEADER + "\n", "no table rows"),
    (HEADER + "\n20,1.0,10,0.1,0.2,0.3,1.4\n", r"\(0, 1\)"),
    (HEADER + "\n20,1.0,ten,0.1,0.2,0.3,0.4\n", "line 2"),
    ("# replicates=many\n" + HEADER + "\n20,1.0,10,0.1,0.2,0.3,0.4\n", "bad replicates"),
    (HEADER + "\n0,1.0,10,0.1,0.2,0.3,0.4\n", "bad k_support"),
])
def test_format_errors(tmp_path, text, match):
    path = tmp_path / "bad.csv"
    path.write_text(text)
    with pytest.raises(TableFormatError, match=match):
        load_table(path)


def test_cli_usage_errors_exit_2(tmp_path, capsys):
    out = str(tmp_path / "x.csv")
    assert cli.main(["simulate", "--n", "10", "--gamma", "0.5", "--k", "inf", "--seed", "1", "--out", out]) == 2
    assert "the unbounded model needs gamma >= 1.05" in capsys.readouterr().err
    assert cli.main(["simulate", "--n", "10", "--gamma", "0.0", "--k", "20", "--seed", "1", "--out", out]) == 2
    assert "simulation needs gamma > 0" in capsys.readouterr().err
    assert cli.main(["simulate", "--n", "10", "--gamma", "1.5", "--k", "20", "--seed", "1", "--out", out,
                     "--quantiles", "0.9,0.95"]) == 2
    assert "schema stores exactly the levels" in capsys.readouterr().err
    with pytest.raises(SystemExit):
        cli.main(["simulate", "--n", "ten", "--gamma", "1.5", "--k", "20", "--out", out])
    assert not os.path.exists(out)
