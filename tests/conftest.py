import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built_artifacts():
    import __graft_entry__ as ge

    ge.build_oracle()
    try:
        ge.build_native()
    except Exception:
        # the CPU suite only needs the library for the symbol checks, which report it
        pass
    yield


@pytest.fixture
def paths():
    """Force planner choices (obt_set_path_option) for one test: ``paths(wide=1, fan=0)``;
    the previous values are restored afterwards."""
    from paper_2211_00391_b200 import _native

    saved = {}

    def force(**opts):
        for k, v in opts.items():
            if k not in saved:
                saved[k] = _native.get_path_option(k)
            _native.set_path_option(k, v)

    yield force
    for k, v in saved.items():
        _native.set_path_option(k, v)
