// FP64 SIPDG operator kernels for sm_100a (B200).  Included by ipdg.cu only.
//
// Paper: arXiv:1801.00246, P:n = PAPER.md line n.
//
// Formulation (exactly equal to Eqs. ellipticOp1/ellipticOp3, on affine
// elements):
//   u_r = Dr u, u_s = Ds u                                   (Alg. AxG)
//   delta_f = u+ - u- at the face nodes                       (jump; traces P:553-554)
//   w_r = J(G_rr u_r + G_rs u_s),  w_s = J(G_rs u_r + G_ss u_s),  G = [r_x s_x; r_y s_y]
//   g_f = 1/2 n.(grad u- + grad u+) + tau_f delta_f          (SIPDG flux, Eq. INS_SD_5)
//   Au  = Sr^T w_r + Ss^T w_s                                 (volume, S = M D)
//       + sum_f (LIFT_f^T Sr)^T (1/2 sJ_f (r_x n_x + r_y n_y) delta_f)   (lift of the jump,
//       + sum_f (LIFT_f^T Ss)^T (1/2 sJ_f (s_x n_x + s_y n_y) delta_f)    P:454-458)
//       - sum_f sJ_f scatter_{Fmask_f}(M1D g_f)               (surface flux x face mass)
//       + lambda J M u                                        (Eq. ellipticOp1)
// Every dense contraction over many elements runs on the FP64 tensor cores
// (DMMA, mma.sync.m8n8k4.f64; tcgen05 has no f64 kind): the element index is the
// M dimension (8 elements per MMA row block), node indices are N and K.  The
// operator tables are staged once per persistent CTA in shared memory in
// fragment-major order, so every B-fragment load is one conflict-free LDS.64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ipdg {

template <int N_>
struct Tr {
  static constexpr int N = N_;
  static constexpr int NP = (N + 1) * (N + 2) / 2;
  static constexpr int NFP = N + 1;
  static constexpr int NF3 = 3 * NFP;
  static constexpr int NPK = (NP + 3) / 4 * 4;   // K extent of u (grad GEMM)
  static constexpr int NPN = (NP + 7) / 8 * 8;   // N extent of node outputs
  static constexpr int NT = NPN / 8;             // n-tiles per node field
  static constexpr int KCG = NPK / 4;            // k-chunks, grad GEMM
  static constexpr int NF3P = (NF3 + 3) / 4 * 4;   // face nodes padded to whole k-chunks
  static constexpr int NQ = NF3P / 4;               // face-node passes of the 4 lanes of an element
  static constexpr int KF = 3 * NF3P;               // K extent of the face block (a_r delta | a_s delta | -sJ g)
  static constexpr int KCW = 4 * NT;             // k-chunks fed from registers (w_r, w_s in C layout)
  static constexpr int KCF = KF / 4;             // k-chunks of the face block (fed from registers)
  static constexpr int KCM = NPK / 4;            // k-chunks of the lambda (mass) block
  static constexpr int pad416(int s) { return (s % 16 == 4 || s % 16 == 12) ? s : pad416(s + 1); }
  static constexpr int SU = pad416(NPK);         // smem row stride of u (conflict-free A loads)
  static constexpr int SF = pad416(KF);          // smem row stride of the face block
  static constexpr int SXY = 2 * NPN + 2;        // smem row stride of (w_r | w_s) per slot (= 2 mod 16: gathers spread over banks)
  static constexpr int SG = 8;                   // per-slot geometry: rx sx ry sy J det - -
  static constexpr int RPW = NP >= 32 ? 1 : 32 / NP;  // element rows copied per warp pass
  static constexpr int NPASS = (NP + 31) / 32;        // lane passes per row (NP > 32)
  // fragment-table sizes (doubles): [chunk][ntile][lane]
  static constexpr int TAB_G = KCG * 2 * NT * 32;
  static constexpr int TAB_M = (KCW + KCF) * NT * 32;
  static constexpr int TAB_L = KCM * NT * 32;
  // launch shape: W warps, one own 8-element tile per warp
  static constexpr int W = N >= 7 ? 4 : 8;
  static constexpr int E = 8 * W;
  static constexpr int MINB = N <= 5 ? 2 : 1;
  static constexpr int FGS = E + 8;              // field stride of the per-face geometry (bank spread, see P2)  // CTAs per SM the register allocation must allow
};

// Face-node index in closed form for the row-by-row node order (refops.cpp; verified at setup):
// row j (s index) holds N+1-j nodes starting at off(j) = j(N+1) - j(j-1)/2.
//   face 0 (s = -1):   node k            face 1 (r+s = 0): node off(k) + N - k
//   face 2 (r = -1):   node off(k)
template <int N>
__host__ __device__ __forceinline__ constexpr int fmask_cf(int f, int k) {
  return f == 0 ? k : (f == 1 ? k * (N + 1) - (k * (k - 1)) / 2 + N - k : k * (N + 1) - (k * (k - 1)) / 2);
}

// per-element face record length (k_geofacs) in doubles: 9 used, padded to 10 so a block's records
// (80 B each) are a 16-byte multiple for a bulk copy
constexpr int kGF = 10;

// k_gather: threads per CTA (one element per thread)
constexpr int kGatherThreads = 128;

// Kernel parameters (plain pointers; all device memory).
struct AxArgs {
  int64_t K;             // local elements
  int64_t H;             // halo ghosts (rows of halo_p)
  int nblocks;           // element blocks (contiguous ranges of <= E own elements)
  const int* blist;      // k_pipe: null = all blocks, else process blocks blist[0..nlist) (split pass A)
  int nlist;
  int red_part;          // k_pipe PCG: 0 = p.Ap -> red_A; 1 = -> red_A_part; 2 = red_A = red_A_part + own
  const int* boff;       // [nblocks+1] first element of each block
  const double4* geo;    // [K + H] r_x, s_x, r_y, s_y  (H = halo ghosts, multi-GPU)
  const short4* nbr;     // [K] per face: slot (x,y,z), w = flags: face f -> bits 4f..4f+3 = (f' | bc << 2)
  const int4* nbg;       // [K] neighbour element per face (>= K: halo ghost; self on boundary) + the same flags (k_gather)
  const int* goff;       // [nblocks+1] ghost list offsets
  const int* gid;        // ghost element ids (>= K: halo index K + h)
  const double* tables;  // fragment tables: G | M | L
  const double4* gG;     // [K + H] (J G_rr, J G_rs, J G_ss, J) per element (k_pipe)
  const double* gF;      // [K][kGF = 10] per face (1/2 sJ n.grad r, 1/2 sJ n.grad s, sJ tau) (k_pipe, k_gather)
  double tau_c;          // (N+1)(N+2)/2 * tau_scale
  double lambda;
  // MODE_AX
  const double* u;       // [K] x NP
  double* Au;
  // MODE_PCG_A
  const double* r;
  const double* dinv;    // null: no preconditioner
  const double* z;       // z = D^-1 r (written by pass B / init), = r without preconditioner
  double* p_even;        // p_k lives in p_even when k is even, p_odd when k is odd
  double* p_odd;         //   (double buffer: ghosts read p_{k-1} while owners write p_k)
  double* x;             // deferred update x += alpha_{k-1} p_{k-1}
  int defer_x;           // k_pipe: 1 = pass A applies the deferred x update, 0 = pass B updates x
  const double* halo_p;  // [H x NP] received ghost values of p_k (multi-GPU), else null
  struct PcgState* st;
  double* partials;      // [gridDim.x]
  unsigned int* counter;
  // k_tpb (thread per element, blocks of tpb_e(N) consecutive elements)
  const short4* nbt;     // [K] per face: slot (own e - e0 < E, ghost face E + g with E = tpb_e(N), boundary: own) + flags as nbr
  const int* gfoff;      // [nblocks_t + 1] ghost-face list offsets
  const int* gface;      // ghost faces: (neighbour element << 2) | its face, sorted by face within a block
  const double* tauF;    // [K x 3] sJ tau per face
};

// k_tpb: elements per CTA (block of consecutive elements)
#ifndef IPDG_TPB_E
#define IPDG_TPB_E 128
#endif
constexpr int kTpbE = IPDG_TPB_E;
// elements per k_tpb block (= threads per CTA) by degree: 256 at N = 4 (two 100 KB CTAs per SM; fewer ghost
// faces per element; pass A 75.4 vs 77.3 us on C2, profiles/r02d_tpb_block_size.txt), kTpbE elsewhere
// (N = 5 would not fit twice per SM)
#ifndef IPDG_TPB_BIGE
#define IPDG_TPB_BIGE (1 << 4)  // degrees (bit N) with 2 kTpbE-element blocks
#endif
__host__ __device__ constexpr int tpb_e(int N) { return ((IPDG_TPB_BIGE >> N) & 1) ? 2 * kTpbE : kTpbE; }

// Device-side PCG state (one per context).  See ipdg.cu "PCG protocol".
struct PcgState {
  double rho_hist[4];  // rho_k = r_k . z_k at slot k & 3 (global values)
  double red_A;        // sigma_k = p_k . A p_k  (pass-A output, all-reduced in place)
  double red_A_part;   // first half of a split pass A (interior blocks)
  double red_B[3];     // (rho_k, rr_k, bb) pass-B / init output, all-reduced in place
  double bb;           // ||b||^2
  double tol2;         // tol^2
  double final_rr;
  long long it;        // completed iterations
  long long maxit;
  long long stop_iter; // -1 while running
  int status;          // 0 ok, 1 not converged, -4 breakdown
  int precond;
};

}  // namespace ipdg
