// Reference operators in __constant__ memory for the thread-per-element kernels (N <= 4): k_gather
// (sipdg_gather.cuh) and k_dgop_tpe (dgops.cuh).  Every DFMA takes its operator entry as a
// compile-time index into c_tpe<N> (a uniform constant-bank operand): no shared-memory traffic.
// Paper: arXiv:1801.00246; formulation in kernels.cuh.
#pragma once
#include "kernels.cuh"

namespace ipdg {

template <int N_>
struct TrT {
  static constexpr int N = N_;
  static constexpr int NP = (N + 1) * (N + 2) / 2, NFP = N + 1, NF3 = 3 * NFP;
  // __constant__ table layout (doubles)
  static constexpr int O_DR = 0, O_DS = NP * NP, O_SR = 2 * NP * NP, O_SS = 3 * NP * NP;
  static constexpr int O_LSR = 4 * NP * NP;             // [fk][n]: (LIFT^T Sr)[fk][n]
  static constexpr int O_LSS = O_LSR + NF3 * NP;
  static constexpr int O_M1D = O_LSS + NF3 * NP;       // [k][m]
  static constexpr int O_M = O_M1D + NFP * NFP;         // [n][j] reference mass (lambda term)
  static constexpr int O_LIFT = O_M + NP * NP;          // [n][fk] LIFT (DG gradient / divergence, dgops.cuh)
  static constexpr int TOTAL = O_LIFT + NP * NF3;
};

template <int N>
__constant__ double c_tpe[TrT<N>::TOTAL];

}  // namespace ipdg
