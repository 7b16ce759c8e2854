"""CPU: the C-ABI libraries load and export every entry point include/tmgx.h declares."""
import os
import re

import pytest

from paper_1604_07163_b200 import tmgx as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "tmgx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tmgx_[a-z0-9_]+)\s*\(", src)))


@pytest.mark.parametrize("parity", [False, True])
def test_exports(parity):
    L = T.load(parity)
    names = declared()
    assert set(names) == set(T.EXPORTS)
    for n in names:
        assert hasattr(L, n), n
    assert L.tmgx_parity_build() == (1 if parity else 0)


def test_errors_map_to_exceptions():
    with pytest.raises(T.ConfigError):
        T.create_grid_header(8, (4, 4, 4), hint=(8, 1, 1))
    with pytest.raises(T.ConfigError):
        T.split_strided(4, 0)
    with pytest.raises(T.ConfigError):
        T.coarsen(T.create_grid_header(1, (8, 8, 8)))
