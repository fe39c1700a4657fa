"""Run the reference's own unit-test modules against the drop-in.

The reference's tests import ``zipfks``; this tool writes a throwaway shim package ``zipfks``
into a temporary directory whose modules ARE this package's modules (``sys.modules`` aliases:
zipfks.distribution -> paper_1305_6738_b200.distribution, ..., zipfks.observations and
zipfks.reporting -> paper_1305_6738_b200.bespoke, ``python -m zipfks`` -> our CLI), then runs
pytest on a directory holding the reference's test files.  Nothing of the reference is
imported: every call the tests make lands in this package (and so on the GPU).

    python tools/run_reference_tests.py --tests /path/to/copy/of/pkg/tests [-- pytest args]

The reference tree does not travel to the GPU box: copy pkg/tests into a git-ignored
directory of the repo for one gpurun call and delete it afterwards.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SHIM_INIT = '''"""Test shim: ``zipfks`` resolved to paper_1305_6738_b200 (tools/run_reference_tests.py)."""
import sys

import paper_1305_6738_b200 as _impl
from paper_1305_6738_b200 import *  # noqa: F401,F403
from paper_1305_6738_b200 import (bespoke, cli, distribution, estimate, gof, montecarlo, series,  # noqa: F401
                                  tablefile)

__version__ = "1.0.0"
for _name, _mod in {"distribution": distribution, "estimate": estimate, "gof": gof, "montecarlo": montecarlo,
                    "series": series, "tablefile": tablefile, "cli": cli, "observations": bespoke,
                    "reporting": bespoke}.items():
    sys.modules[f"zipfks.{_name}"] = _mod
    globals()[_name] = _mod
observations = bespoke
reporting = bespoke
'''
SHIM_MAIN = '''import sys

from paper_1305_6738_b200.cli import main

sys.exit(main())
'''


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tests", required=True, help="directory holding the reference's test modules")
    ap.add_argument("pytest_args", nargs="*")
    args = ap.parse_args()
    with tempfile.TemporaryDirectory() as tmp:
        pkg = os.path.join(tmp, "zipfks")
        os.makedirs(pkg)
        with open(os.path.join(pkg, "__init__.py"), "w") as fh:
            fh.write(SHIM_INIT)
        with open(os.path.join(pkg, "__main__.py"), "w") as fh:
            fh.write(SHIM_MAIN)
        env = dict(os.environ, PYTHONPATH=os.pathsep.join([tmp, ROOT, os.environ.get("PYTHONPATH", "")]))
        cmd = [sys.executable, "-m", "pytest", args.tests, "-p", "no:cacheprovider", "-rfE", *args.pytest_args]
        print(" ".join(cmd), flush=True)
        return subprocess.run(cmd, env=env, cwd=tmp).returncode


if __name__ == "__main__":
    sys.exit(main())
