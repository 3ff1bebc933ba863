"""CPU-side checks of the C ABI: the library loads, exports every symbol include/ljmd.h
declares, host-only planning calls work, and compute calls fail loudly without a GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1704_03329_b200 import build, ljmd
    build.build()
    return ljmd.load()


def declared():
    src = open(os.path.join(ROOT, "include", "ljmd.h")).read()
    return sorted(set(re.findall(r"\b(ljmd_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    from paper_1704_03329_b200 import ljmd
    names = declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(ljmd.EXPORTS)


def test_version(lib):
    from paper_1704_03329_b200 import version
    assert "sm_100a" in version()


def test_plan_cells_matches_oracle(lib, orc):
    from paper_1704_03329_b200 import plan_cells
    for L in ([16.795961913825] * 3, [107.494156248480] * 3, [8.5, 9.0, 33.0], [10.0, 10.0, 10.0]):
        assert plan_cells(L, 2.75).tolist() == orc.cell_dims(L, 2.75).tolist()
    assert plan_cells([9.0, 9.0, 9.0], 2.75).tolist() == [3, 3, 3]       # SPEC.md:178-180 style
    assert plan_cells([10.0] * 3, 2.5).tolist() == [3, 3, 3]              # 10/(2.5(1+1e-12)) < 4 (safety factor)
    with pytest.raises(Exception):
        plan_cells([8.0, 9.0, 9.0], 2.75)


def test_plan_slab_partition():
    from paper_1704_03329_b200 import plan_slab
    for ncz, p in ((78, 8), (78, 1), (156, 8), (39, 2), (5, 5)):
        spans = [plan_slab(ncz, p, r) for r in range(p)]
        assert spans[0][0] == 0 and spans[-1][1] == ncz
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    assert [plan_slab(78, 8, r)[1] - plan_slab(78, 8, r)[0] for r in range(8)] == [10, 10, 10, 10, 10, 10, 9, 9]


def test_no_cpu_fallback(lib):
    """Without a GPU the engine refuses to compute (no silent host path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1704_03329_b200 import LJMD, LjmdError
    with pytest.raises(LjmdError, match="CUDA"):
        LJMD(np.zeros((4, 3)), np.zeros((4, 3)), [10.0, 10.0, 10.0])


def test_product_does_not_import_oracle():
    """The product package shares no code with oracle/ (independence rule)."""
    pkg = os.path.join(ROOT, "paper_1704_03329_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dp, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "ljmd_oracle" not in s, f
