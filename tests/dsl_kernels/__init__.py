"""The paper's C kernels (verbatim up to the sign reading R1), shared by the oracle pins and
the GPU DSL parity tests: they are the *input* of a pair loop, like a particle array."""

# Listing lst:LJ-kernel; constants sigma2, rc_sq, CV = 4 eps, CF = +48 eps/sigma^2
# (reading R1: the listing's caption has -48, but F.i += f_tmp * (r_i - r_j) must be repulsive
# at short range)
LJ = """
const double dr0 = r.i[0] - r.j[0];
const double dr1 = r.i[1] - r.j[1];
const double dr2 = r.i[2] - r.j[2];
// Calculate squared distance
// dr2 = |r_i - r_j|^2
double dr_sq = dr0*dr0+dr1*dr1+dr2*dr2;
// (sigma/dr)^2
const double r_m2 = sigma2/dr_sq;
// (sigma/dr)^4
const double r_m4 = r_m2*r_m2;
// (sigma/dr)^6
const double r_m6 = r_m4*r_m2;
// (sigma/dr)^8
const double r_m8 = r_m4*r_m4;
// Increment potential energy
u[0]+= (dr_sq<rc_sq) ? CV*((r_m6-1.0)*r_m6+0.25) : 0.0;
const double f_tmp=CF*(r_m6-0.5)*r_m8;
// Increment forces
F.i[0]+= (dr_sq<rc_sq)?f_tmp*dr0:0.0;
F.i[1]+= (dr_sq<rc_sq)?f_tmp*dr1:0.0;
F.i[2]+= (dr_sq<rc_sq)?f_tmp*dr2:0.0;
"""

LJ_CONSTANTS = {"sigma2": 1.0, "rc_sq": 6.25, "CV": 4.0, "CF": 48.0}

# Listing lst:simple-kernel: Eqs. eqn:simple_op, eqn:simple_op_global
SIMPLE = """
  double da_sq = 0.0;
  for (int r=0;r<dimension;++r) {
    double da = a.i[r]-a.j[r];
    da_sq += da*da;
  }
  b.i[0] += da_sq;
  S += da_sq*da_sq;
"""

# Listings lst:position_update / lst:velocity_update, velocity half of line 6 / 8
VEL_UPDATE = """
v.i[0] += F.i[0]*dht_iMASS;
v.i[1] += F.i[1]*dht_iMASS;
v.i[2] += F.i[2]*dht_iMASS;
"""

# Example 1: kinetic energy as a Particle Loop with a global INC
KINETIC = """
k[0] += 0.5*mass*(v.i[0]*v.i[0] + v.i[1]*v.i[1] + v.i[2]*v.i[2]);
"""

# Listing lst:CNA-kernel_I
CNA_I = """
// Calculate squared distance
const double dr0 = r.i[0] - r.j[0];
const double dr1 = r.i[1] - r.j[1];
const double dr2 = r.i[2] - r.j[2];
double dr_sq = dr0*dr0+dr1*dr1+dr2*dr2;
if (dr_sq < rc_sq) {
  // Add direct bond
  bond.i[2*n_bond.i[0]] = id.i[0];
  bond.i[2*n_bond.i[0]+1] = id.j[0];
  // Increment number of neighbours
  n_nb.i[0]++;
  // Increment number of bonds
  n_bond.i[0]++;
}
"""

# Listing lst:CNA-kernel_II
CNA_II = """
// Calculate squared distance
const double dr0 = r.i[0] - r.j[0];
const double dr1 = r.i[1] - r.j[1];
const double dr2 = r.i[2] - r.j[2];
double dr_sq = dr0*dr0+dr1*dr1+dr2*dr2;
if (dr_sq < rc_sq) {
  for (int k=0;k<n_nb.j[0];++k) {
    // Add indirect bond
    if (bond.j[2*k+1] != id.i[0]) {
      bond.i[2*n_bond.i[0]] = bond.j[2*k];
      bond.i[2*n_bond.i[0]+1] = bond.j[2*k+1];
      // Increment number of bonds
      n_bond.i[0]++;
    }
  }
}
"""
