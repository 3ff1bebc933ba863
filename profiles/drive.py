#!/usr/bin/env python
"""Profiling driver (ncu target): C2 init (one full rebuild), 20 MD steps (one more
rebuild), then the two analyses.  Not a bench: numbers taken under ncu are never reported
as bench values.

usage: ncu --set full -k regex:'k_build_nlist|k_list_rr|k_boa|k_cna' python profiles/drive.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import ljinputs as li  # noqa: E402
from paper_1704_03329_b200 import LJMD  # noqa: E402


def main():
    cfg = li.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    pos, vel, box = cfg.build()
    with LJMD(pos, vel, box) as md:
        md.step(20)
        md.boa(6, 1.5)
        a = li.fcc_lattice_constant()
        md.cna(a * (1.0 / 2 ** 0.5 + 1.0) / 2.0)


if __name__ == "__main__":
    main()
