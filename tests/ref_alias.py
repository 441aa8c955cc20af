"""pytest plugin: run the reference's OWN test files against this package.

Loaded with ``-p ref_alias`` (tests/ on PYTHONPATH) by
tests/test_reference_unmodified.py.  It maps the module ``kvweaver`` and its
hot-path submodules (``kvweaver/__init__.py:12-72``; ``kvweaver.cli``'s CSV
row helpers -> ``report``) onto
``paper_2603_14371_b200`` before the reference test files import them, so
``from kvweaver import ToyBackend, KvManager, run_simulation, ...`` binds the
B200 package: ``ToyBackend`` / ``make_backend("Toy")`` are the CUDA toy
backend over the paged HBM pool, ``KvManager`` / the scheduler / the frame
driver / metrics / workload / rng / verify are this package's.  The test files
themselves come unmodified from the reference install (baseline/_ref/
kvweaver_tests, tools/install_reference.sh).  Out-of-scope reference modules
(config, cli, svg) are not aliased and their tests not run.
"""

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

_SUBMODULES = ("backend", "kv_manager", "metrics", "rng", "scheduler", "sim_engine", "verify", "workload")
# the CSV row helpers the acceptance tests import from the (out-of-scope) CLI
_RENAMED = {"cli": "report"}


def _install() -> None:
    pkg = importlib.import_module("paper_2603_14371_b200")
    sys.modules["kvweaver"] = pkg
    for sub in _SUBMODULES:
        mod = importlib.import_module(f"paper_2603_14371_b200.{sub}")
        sys.modules[f"kvweaver.{sub}"] = mod
        setattr(pkg, sub, mod)
    for ref_name, ours in _RENAMED.items():
        sys.modules[f"kvweaver.{ref_name}"] = importlib.import_module(f"paper_2603_14371_b200.{ours}")


_install()
