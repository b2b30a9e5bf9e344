// Reference-triangle operators of degree N (host side of libipdg).  See refops.cpp.
#pragma once
#include <vector>

namespace ipdg {

struct RefOps {
  int N = 0, Np = 0, Nfp = 0;
  std::vector<double> r, s;          // Np node coordinates on the bi-unit triangle
  std::vector<double> gll;           // Nfp Gauss-Lobatto points
  std::vector<double> Dr, Ds;        // Np x Np, row-major: (Dr u)_i = sum_j Dr[i][j] u_j
  std::vector<double> M;             // Np x Np reference mass (Eq. elMass on the reference element)
  std::vector<double> Sr, Ss;        // M Dr, M Ds
  std::vector<double> M1D;           // Nfp x Nfp face mass on [-1,1]
  std::vector<double> LIFT;          // Np x 3Nfp, M^{-1} E (Eq. elLift)
  std::vector<double> Minv;          // Np x Np, M^{-1} = V V^T (block-Jacobi preconditioner)
  std::vector<int> Fmask;            // 3 x Nfp node ids of each face
};

RefOps build_refops(int N);
// p-multigrid transfer (R23): (fine.Np x coarse.Np) values of the degree-coarse nodal basis at
// the degree-fine nodes, V_c(r_f, s_f) V_c^{-1}
std::vector<double> interp_matrix(const RefOps& fine, const RefOps& coarse);

// Subcycling advection operators (Eq. INS_CUB_N; Alg. SSV / SSS):
// volume cubature = Gauss-Legendre x Gauss-Legendre on the collapsed square with the Duffy factor in the
// weights, face cubature = Gauss-Legendre, both exact to degree 3N.
struct AdvectOps {
  int nc = 0, ncf = 0;               // volume points, points per face
  std::vector<double> I;             // nc x Np: nodal basis at the volume points
  std::vector<double> Pr, Ps;        // Np x nc: M^{-1} w_i (d l_m / dr)(x_i), likewise d/ds
  std::vector<double> If;            // ncf x Nfp: face-node Lagrange basis at the face points (face order)
  std::vector<double> Lc;            // Np x 3 ncf: M^{-1} w_j l_m(x_fj) (cubature lift)
};
AdvectOps build_advect_ops(const RefOps& R);

}  // namespace ipdg
