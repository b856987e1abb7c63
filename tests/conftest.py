import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle():
    """The CPU oracle (plain-C restatement, oracle/gtoracle.c) — the checker."""
    import oracle_lib
    return oracle_lib.load()


@pytest.fixture(scope="session")
def golden():
    return ROOT / "tests" / "golden"


@pytest.fixture(scope="session")
def gt():
    """The product package; its CUDA library must be present (no fallback)."""
    lib = ROOT / "paper_2111_14991_b200" / "libgridtune_b200.so"
    if not lib.exists():
        subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.build_library()"],
                       cwd=str(ROOT), check=True)
    import paper_2111_14991_b200 as m
    m.load()
    return m
