#!/usr/bin/env python
"""Profiling driver (ncu target): C2 init (one full rebuild), 20 MD steps (one more
rebuild), the two analyses, the paper's LJ kernel as a DSL PairLoop, and two steps of the
Newton-3 variant.  Not a bench: numbers taken under ncu are never reported as bench values.

usage: ncu --set full -k regex:'k_build_nlist|k_list_rr|k_boa|k_cna|ljmd_dsl|k_force_half|k_vv' \
           python profiles/drive.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import ljinputs as li  # noqa: E402
from paper_1704_03329_b200 import LJMD, dsl  # noqa: E402

LJ = """
const double dr0 = r.i[0] - r.j[0];
const double dr1 = r.i[1] - r.j[1];
const double dr2 = r.i[2] - r.j[2];
double dr_sq = dr0*dr0+dr1*dr1+dr2*dr2;
const double r_m2 = sigma2/dr_sq;
const double r_m4 = r_m2*r_m2;
const double r_m6 = r_m4*r_m2;
const double r_m8 = r_m4*r_m4;
u[0]+= (dr_sq<rc_sq) ? CV*((r_m6-1.0)*r_m6+0.25) : 0.0;
const double f_tmp=CF*(r_m6-0.5)*r_m8;
F.i[0]+= (dr_sq<rc_sq)?f_tmp*dr0:0.0;
F.i[1]+= (dr_sq<rc_sq)?f_tmp*dr1:0.0;
F.i[2]+= (dr_sq<rc_sq)?f_tmp*dr2:0.0;
"""


def main():
    cfg = li.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
    pos, vel, box = cfg.build()
    with LJMD(pos, vel, box) as md:
        md.step(20)
        md.boa(6, 1.5)
        a = li.fcc_lattice_constant()
        md.cna(a * (1.0 / 2 ** 0.5 + 1.0) / 2.0)
        F, u = dsl.ParticleDat(md, ncomp=3), dsl.ScalarArray(md)
        consts = tuple(dsl.Constant(k, v) for k, v in
                       {"sigma2": 1.0, "rc_sq": li.RC ** 2, "CV": 4.0, "CF": 48.0}.items())
        dsl.PairLoop(dsl.Kernel("lj", LJ, consts),
                     {"r": dsl.PositionDat(md)(dsl.READ), "F": F(dsl.INC_ZERO), "u": u(dsl.INC_ZERO)},
                     shell_cutoff=li.RC).execute()
    with LJMD(pos, vel, box, newton3=1) as md:
        md.step(2)


if __name__ == "__main__":
    main()
