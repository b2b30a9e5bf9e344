// libipdg context, error macros and the per-degree dispatch table (shared by ipdg.cu and impl_N.cu).
// Paper: arXiv:1801.00246 (P:n = PAPER.md line n).  Design: DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ipdg.h"
#include "refops.h"
#include "kernels.cuh"

using namespace ipdg;

struct ipdg_ctx_s {
  int N = 0, device = 0, sms = 0;
  RefOps ref;
  int64_t K = 0, H = 0;  // local elements, halo ghosts
  double tau_c = 0.0;
  bool has_dirichlet = false;
  // device mesh data
  double4* geo = nullptr;
  double4* gG = nullptr;  // per-element J G^T G records (k_pipe)
  double* gF = nullptr;   // per-face lift coefficients and sJ tau (k_pipe)
  short4* nbr = nullptr;
  int* goff = nullptr;
  int* gid = nullptr;
  int* boff = nullptr;
  int* etoe = nullptr;
  int8_t* bcode = nullptr;
  double* vxy = nullptr;
  double* rs = nullptr;
  double* Mref = nullptr;
  double* Minv = nullptr;  // M^{-1} (block-Jacobi preconditioner)
  double* dgops = nullptr; // Dr | Ds | LIFT (DG gradient / divergence)
  double* tables = nullptr;
  double* diagtab = nullptr;
  int nblocks = 0, gmax = 0;
  int E = 0;
  // split variant (k_grad + k_flux): neighbour ids per element, W = [w_r | w_s] scratch
  int4* nbg = nullptr;
  double* W2 = nullptr;
  // thread-per-element block variant (k_tpb): kTpbE consecutive elements per block, ghost faces
  short4* nbt = nullptr;
  int* gfoff_t = nullptr;
  int* gface_t = nullptr;
  double* tauF = nullptr;
  int nblocks_t = 0, gmax_t = 0;
  int* blist_t = nullptr;      // split pass A: [interior blocks | halo-boundary blocks]
  int nbt_split[2] = {0, 0};
  size_t smem_tpb_m[2] = {0, 0};  // [mode]
  bool tpb_ok[2][2] = {{false, false}, {false, false}};  // [mode][lam] fits on an SM
  int tpb_grid[2][2] = {{0, 0}, {0, 0}};  // [mode][lam] persistent grid: resident CTAs per SM x SMs
  // p-multigrid preconditioner (IPDG_PRECOND_PMG; pmg.cuh, R22-R25): level 0 is this context,
  // levels 1.. are child contexts of degree d_l on the same mesh
  struct PmgLevel {
    ipdg_ctx ctx = nullptr;   // child context (level 0: null, the parent)
    int N = 0, Np = 0;
    double lmax = 0.0;
    double* buf = nullptr;    // dinv | b | x | r | d | t | y, K*Np each (256-byte aligned)
    int64_t seg = 0;          // doubles per vector
    double* I = nullptr;      // prolongation from level l+1 (Np x Np_{l+1}, row-major), device
  };
  std::vector<PmgLevel> pmg;
  double pmg_lambda = -1.0;
  PcgState* pmg_gate = nullptr;   // PCG state that gates the cycle's vector kernels (null: ipdg_pmg_apply)
  std::vector<int32_t> pend_etov;  // mesh kept for the child contexts
  double tau_scale = 1.0;
  double* adv_tab = nullptr;  // advection operators I | Pr | Ps | If | Lc (build_advect_ops), built on first use
  int grid_cap = 0;  // debug: cap on every persistent grid (0 = off)
  int variant = 0;  // 0 auto, 1 fused, 2 split, 3 thread-per-element (N <= 4), 4 pipelined fused
  // pipelined fused variant (k_pipe): same schedule as k_sipdg; grid 0 = does not fit
  size_t smem_pipe[2][2] = {{0, 0}, {0, 0}};
  int grid_pipe[2][2] = {{0, 0}, {0, 0}};
  bool pipe_xb[2] = {false, false};  // [lam]: k_pipe's pass A leaves x to pass B (no room for x staging)
  size_t smem_grad = 0, smem_flux[2] = {0, 0};
  int grid_grad = 0, grid_flux[2][2] = {{0, 0}, {0, 0}};
  size_t smem[2][2] = {{0, 0}, {0, 0}};  // [mode][lam]
  int grid[2][2] = {{0, 0}, {0, 0}};  // [mode][lam]
  // host copies for introspection
  std::vector<int> etoe_h, etof_h;
  // PCG
  PcgState* st = nullptr;
  PcgState* st_host = nullptr;
  double* partials = nullptr;
  int partials_cap = 0;  // slots per reduced quantity
  unsigned int* counter = nullptr;
  void* ws = nullptr;
  int64_t ws_bytes = 0;
  bool ws_owned = false;
  double* hostio = nullptr;  // ipdg_pcg_solve_host: device copies of b | x (hostio_n doubles each)
  int64_t hostio_n = 0;
  double *r = nullptr, *pe = nullptr, *po = nullptr, *Ap = nullptr, *dinv = nullptr, *zb = nullptr;
  double dinv_lambda = -1.0;
  bool dinv_valid = false;
  // current solve
  double* x = nullptr;
  double lambda = 0.0;
  int precond = 0;
  bool xb = false;  // pass B updates x (k_pipe pass A); else pass A applies the deferred update
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};  // [0]: 1 iteration, [1]: kChunk iterations
  const void* gkey_x = nullptr;
  double gkey_lambda = -1.0;
  int gkey_precond = -1;
  cudaStream_t cap_stream = nullptr;
  // split pass A (k_pipe): interior blocks, then halo-boundary blocks once the exchange (on comm_stream)
  // has landed -- the halo exchange overlaps the interior work
  bool split_a = false;        // multi-GPU halo, or forced for tests (ipdg_debug_split_pass_a)
  int force_split = 0;
  int* blist = nullptr;        // [interior block ids | boundary block ids]
  int nb_split[2] = {0, 0};
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_halo = nullptr;
  bool halo_ev_pending = false;
  // pending host mesh (ipdg_upload_mesh -> ipdg_upload_halo)
  int64_t pend_K = 0, pend_remote = 0;
  std::vector<int> pend_etoe, pend_etof;
  std::vector<int8_t> pend_bc;
  std::vector<double> pend_vxy, pend_VX, pend_VY;
  // halo (multi-GPU): S sent element rows, H received ghost rows
  int64_t S = 0;
  int* send_idx = nullptr;
  double* sendbuf = nullptr;
  double* halobuf = nullptr;
  std::vector<int> nbr_rank;
  std::vector<int64_t> send_off, recv_off;
  bool has_dirichlet_global = false;
  bool halo_external = false;  // caller fills the halo buffer (ipdg_halo_set), no NCCL
  // multi-GPU
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  std::string err;
  int64_t launches = 0;
  int launches_per_iter = 2;  // kernels per PCG iteration (set when the iteration graph is captured)
};

static constexpr int kChunk = 32;
static constexpr int kCommSlots = 8;  // CTA slots left free for NCCL during an overlapped pass

#define FAIL(ctx, code, ...)                                         \
  do {                                                              \
    char b_[512];                                                   \
    snprintf(b_, sizeof(b_), __VA_ARGS__);                          \
    if (ctx) (ctx)->err = b_;                                        \
    return code;                                                    \
  } while (0)
#define CUDA_TRY(ctx, x)                                                                            \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) FAIL(ctx, IPDG_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define NCCL_TRY(ctx, x)                                                                           \
  do {                                                                                             \
    ncclResult_t r_ = (x);                                                                         \
    if (r_ != ncclSuccess) FAIL(ctx, IPDG_ENCCL, "%s: %s", #x, ncclGetErrorString(r_));            \
  } while (0)

#define TRY(x)                 \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != IPDG_OK) return rc_; \
  } while (0)

template <class Tp>
static int upload(ipdg_ctx c, Tp** dst, const Tp* src, size_t n) {
  if (*dst) cudaFree(*dst);
  *dst = nullptr;
  CUDA_TRY(c, cudaMalloc((void**)dst, std::max<size_t>(n, 1) * sizeof(Tp)));
  if (n) CUDA_TRY(c, cudaMemcpy(*dst, src, n * sizeof(Tp), cudaMemcpyHostToDevice));
  return IPDG_OK;
}


// per-degree implementation (impl.cuh, one translation unit per N: impl_N.cu)
struct ImplOps {
  std::vector<double> (*build_tables)(const RefOps&);
  std::vector<double> (*build_diagtab)(const RefOps&);
  int (*configure)(ipdg_ctx);
  int (*resolve)(ipdg_ctx, int, bool, const void*);
  int (*ax)(ipdg_ctx, const double*, double*, double, cudaStream_t);
  int (*pass_a)(ipdg_ctx, cudaStream_t);
  int (*pass_b_bj)(ipdg_ctx, bool, const double*, cudaStream_t);
  int (*dgop)(ipdg_ctx, bool, const double*, const double*, double*, double*, cudaStream_t);
  int (*diag)(ipdg_ctx, double*, double, cudaStream_t);
  int (*mass)(ipdg_ctx, const double*, double*, cudaStream_t);
  int (*upload_constants)(ipdg_ctx);
  int (*advect)(ipdg_ctx, const double* const*, double* const*, cudaStream_t);
};
const ImplOps* impl_ops(int N);
