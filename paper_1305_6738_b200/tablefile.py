"""Cutoff-table CSV files: the on-disk form of ``build_table``'s result.

Byte-compatible with the reference writer and reader (``tablefile.py:31-50`` write,
``tablefile.py:53-135`` load), so a table regenerated on the GPU drops into any consumer of
the reference's ``load_table``::

    # replicates=<R>
    # repetitions=<P>
    # seed=<S>
    k_support,gamma,n,q90,q95,q99,q999
    <K or inf>,<repr(gamma)>,<n>,<repr(q90)>,<repr(q95)>,<repr(q99)>,<repr(q999)>

Rows are gamma-major in the table's grid order; floats use ``repr`` so values round-trip
exactly.  Host-only code: nothing here touches the device.
"""
from __future__ import annotations

import os
from typing import Iterator

from .distribution import Support
from .montecarlo import DEFAULT_LEVELS, CutoffTable

COLUMNS = ("k_support", "gamma", "n", "q90", "q95", "q99", "q999")
_HEADER_LINE = ",".join(COLUMNS)
_META_KEYS = ("replicates", "repetitions", "seed")


class TableFormatError(ValueError):
    """The file does not parse back into a cutoff table (``tablefile.py:23-24``)."""


def _label(support: Support) -> str:
    return "inf" if support.k is None else str(support.k)


def _lines(table: CutoffTable) -> Iterator[str]:
    meta = (table.replicates, table.repetitions, table.base_seed)
    for key, value in zip(_META_KEYS, meta):
        yield f"# {key}={value}"
    yield _HEADER_LINE
    label = _label(table.support)
    for gamma in table.gammas:
        for n in table.ns:
            fields = [label, repr(gamma), str(n)]
            fields.extend(repr(c) for c in table.cells[(gamma, n)])
            yield ",".join(fields)


def format_table(table: CutoffTable) -> str:
    """The file's full text (what ``write_table`` writes)."""
    if table.levels != DEFAULT_LEVELS:
        raise TableFormatError(f"the table file schema holds levels {DEFAULT_LEVELS}, got {table.levels}")
    return "".join(line + "\n" for line in _lines(table))


def write_table(table: CutoffTable, path: str | os.PathLike) -> None:
    """Serialise ``table``; only the standard four quantile levels fit the schema."""
    text = format_table(table)
    with open(path, "w", encoding="utf-8") as out:
        out.write(text)


def _parse_row(path, line_no: int, line: str) -> tuple[str, float, int, tuple[float, ...]]:
    parts = line.split(",")
    if len(parts) != len(COLUMNS):
        raise TableFormatError(f"{path}: line {line_no}: expected {len(COLUMNS)} columns")
    try:
        gamma, n = float(parts[1]), int(parts[2])
        cutoffs = tuple(map(float, parts[3:]))
    except ValueError as err:
        raise TableFormatError(f"{path}: line {line_no}: {err}") from err
    if any(hi < lo for lo, hi in zip(cutoffs, cutoffs[1:])):
        raise TableFormatError(f"{path}: line {line_no}: quantile columns must be nondecreasing")
    if not all(0.0 < c < 1.0 for c in cutoffs):
        raise TableFormatError(f"{path}: line {line_no}: cutoffs must lie in (0, 1)")
    return parts[0], gamma, n, cutoffs


def _support_of(path, labels: set[str]) -> Support:
    if len(labels) != 1:
        raise TableFormatError(f"{path}: mixed k_support values {sorted(labels)}")
    (label,) = labels
    if label == "inf":
        return Support.unbounded()
    try:
        return Support.finite(int(label))
    except ValueError as err:
        raise TableFormatError(f"{path}: bad k_support {label!r}: {err}") from err


def load_table(path: str | os.PathLike) -> CutoffTable:
    """Inverse of ``write_table`` with the reference's format checks and messages."""
    meta: dict[str, int] = {}
    rows = []
    have_header = False
    with open(path, "r", encoding="utf-8") as src:
        for line_no, raw in enumerate(src, start=1):
            line = raw.strip()
            if not line:
                continue
            if line[0] == "#":
                key, _, value = (s.strip() for s in line[1:].partition("="))
                if key in _META_KEYS:
                    try:
                        meta[key] = int(value)
                    except ValueError as err:
                        raise TableFormatError(f"{path}: line {line_no}: bad {key}") from err
            elif have_header:
                rows.append(_parse_row(path, line_no, line))
            elif line == _HEADER_LINE:
                have_header = True
            else:
                raise TableFormatError(f"{path}: line {line_no}: header must be exactly {_HEADER_LINE!r}")
    if not have_header:
        raise TableFormatError(f"{path}: missing header line {_HEADER_LINE!r}")
    if not rows:
        raise TableFormatError(f"{path}: no table rows")
    support = _support_of(path, {r[0] for r in rows})
    # grid axes in first-seen order (dict keys keep insertion order)
    gammas = tuple(dict.fromkeys(r[1] for r in rows))
    ns = tuple(dict.fromkeys(r[2] for r in rows))
    cells: dict[tuple[float, int], tuple[float, ...]] = {}
    for _, gamma, n, cutoffs in rows:
        if (gamma, n) in cells:
            raise TableFormatError(f"{path}: duplicate cell (gamma={gamma}, n={n})")
        cells[(gamma, n)] = cutoffs
    missing = [(g, n) for g in gammas for n in ns if (g, n) not in cells]
    if missing:
        raise TableFormatError(f"{path}: incomplete grid, missing cells {missing[:4]}")
    return CutoffTable(support=support, levels=DEFAULT_LEVELS, gammas=gammas, ns=ns, cells=cells,
                       replicates=meta.get("replicates", 0), repetitions=meta.get("repetitions", 0),
                       base_seed=meta.get("seed", 0))
