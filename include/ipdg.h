/*
 * ipdg.h -- C ABI of libipdg.so: FP64 matrix-free SIPDG Poisson operator and
 * Jacobi-preconditioned CG on affine nodal triangles, for NVIDIA B200 (sm_100a).
 *
 * Paper: Karakus, Chalmers, Swirydowicz, Warburton, "GPU Acceleration of a
 * High-Order Discontinuous Galerkin Incompressible Flow Solver", arXiv:1801.00246.
 * "P:n" below = line n of that paper's LaTeX.
 *
 *   A u ~ -Laplace(u) + lambda u        Eq. ellipticOp1, positive operator
 *   SIPDG Laplacian                     Eq. INS_SD_5
 *   penalty tau^{ef}                    Eq. Ch2.PenaltyParameter
 *   jump [[u]] = u+ - u-, average {u}   Eq. AverageJumpScalar
 *   reference operators, affine map     Eqs. elMass..elementOps
 *   PCG                                 P:219 (SPD with the chosen penalty)
 *
 * Conventions (every entry point):
 *   - Degree 1 <= N <= 8.  Np = (N+1)(N+2)/2 nodes per element, Warp & Blend nodes
 *     (P:56), ordered row by row in s with r increasing on the bi-unit triangle
 *     {r,s >= -1, r+s <= 0} (readings R1-R3).
 *   - A nodal field is K x Np float64, element-major, contiguous.
 *   - Functions taking `stream` enqueue asynchronously on that cudaStream_t
 *     (NULL = legacy default stream) and return after enqueueing; device pointers
 *     are caller-owned (e.g. torch CUDA tensors) and must stay alive until the
 *     stream reaches the work.  Host pointers are read during the call only.
 *   - Return value: IPDG_OK (0) or a negative error code (IPDG_NOT_CONVERGED = 1
 *     is a non-fatal status).  ipdg_last_error() gives a one-line detail.
 *   - A context is not thread-safe; use one per host thread / GPU.
 */
#ifndef IPDG_H
#define IPDG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IPDG_OK 0
#define IPDG_NOT_CONVERGED 1 /* maxit reached; stats filled */
#define IPDG_EINVAL (-1)     /* null pointer, K <= 0, tol < 0, lambda < 0, bad code */
#define IPDG_EDEGREE (-2)    /* N outside 1..8 */
#define IPDG_EMESH (-3)      /* J <= 0, non-manifold edge, unmatched interior face */
#define IPDG_EBREAKDOWN (-4) /* p^T A p <= 0 in PCG */
#define IPDG_ESINGULAR (-5)  /* lambda = 0 and no Dirichlet face: A is singular */
#define IPDG_ECUDA (-6)      /* CUDA runtime error */
#define IPDG_ENCCL (-7)      /* NCCL error */
#define IPDG_ESTATE (-8)     /* call order: e.g. ipdg_ax before ipdg_upload_mesh */

/* boundary codes per element face (face f = edge {EToV[e][f], EToV[e][(f+1)%3]}) */
#define IPDG_BC_INTERIOR 0
#define IPDG_BC_DIRICHLET 1 /* homogeneous; mirror u+ = -u-, grad u+ = grad u- */
#define IPDG_BC_NEUMANN 2   /* homogeneous; mirror u+ = u-,  grad u+ = -grad u- */
#define IPDG_BC_REMOTE 3    /* multi-GPU: neighbour owned by another rank (ipdg_upload_halo) */

/* preconditioners for ipdg_pcg_* */
#define IPDG_PRECOND_NONE 0
#define IPDG_PRECOND_JACOBI 1 /* point Jacobi D = diag(A) (R11) */
#define IPDG_PRECOND_BLOCK_JACOBI 2 /* screened Poisson (lambda > 0, else IPDG_EINVAL): the scaled inverse
                                     * mass matrix on each element, (lambda J^e M)^{-1} */
#define IPDG_PRECOND_PMG 3 /* matrix-free p-multigrid V-cycle (P:223-225 pMG levels; DESIGN.md
                              R22-R26): degrees N -> floor(N/2) -> ... -> 1 on the same mesh, nodal
                              interpolation / its transpose between them, degree-2 Chebyshev smoothing
                              of D^-1 A on [lmax/10, 1.1 lmax] (lmax by 20 power iterations); the degree-1
                              level is only smoothed (the paper's AMG tail is out of scope).  One
                              partition only (IPDG_ESTATE with a halo). */

typedef struct ipdg_ctx_s* ipdg_ctx;

typedef struct {
  int64_t iterations;  /* CG iterations performed */
  double rel_residual; /* ||b - A x||_2 / ||b||_2 from the recursively updated residual */
  double bnorm;        /* ||b||_2 (global over ranks) */
  int32_t status;      /* IPDG_OK, IPDG_NOT_CONVERGED or IPDG_EBREAKDOWN */
  int32_t reserved;
  double seconds;      /* host wall time of the solve call (ipdg_pcg_solve*, ipdg_loopback_pcg_solve) */
} ipdg_stats;

/* Create a context for degree N on CUDA device `device`.  Builds the reference
 * operators (Dr, Ds, M, M1D, LIFT, Fmask; Eqs. elMass-elLift) on the host. */
int ipdg_create(ipdg_ctx* out, int N, int device);
int ipdg_destroy(ipdg_ctx ctx);

/* Upload a mesh (HOST arrays, copied).  K local elements, Nv vertices.
 *   VX, VY   [Nv]    vertex coordinates
 *   EToV     [K*3]   counter-clockwise vertex ids (J > 0 required, else IPDG_EMESH)
 *   bc       [K*3]   IPDG_BC_* per element face
 *   tau_scale        1.0 gives tau exactly as Eq. Ch2.PenaltyParameter:
 *                    (N+1)(N+2)/2 * max(1/h-, 1/h+), h = |E|/|dE^f|; boundary faces use h-.
 * Face neighbours are found by matching vertex pairs.  Builds connectivity, the
 * element-block schedule and the geometric factors on the device. */
int ipdg_upload_mesh(ipdg_ctx ctx, int64_t K, int64_t Nv, const double* VX, const double* VY,
                     const int32_t* EToV, const int8_t* bc, double tau_scale);

/* Au = A u (device pointers, K*Np float64 each; in-place not allowed).  lambda >= 0. */
int ipdg_ax(ipdg_ctx ctx, const double* u, double* Au, double lambda, void* stream);

/* d = diag(A) (device, K*Np), computed exactly from the reference operators: the point-Jacobi
 * preconditioner D^{-1} of the BASELINE C4 "Jacobi-PCG" (P:219 PCG; reading R11 -- the paper's
 * own velocity preconditioner is block Jacobi).  Same face/penalty terms as ipdg_ax. */
int ipdg_diag(ipdg_ctx ctx, double* d, double lambda, void* stream);

/* Mu = J^e M u per element (block-diagonal mass, Eq. elementOps). */
int ipdg_mass(ipdg_ctx ctx, const double* u, double* Mu, void* stream);

/* Physical node coordinates x, y (device, K*Np each): x = Phi^e(r,s) (Eq. operators1). */
int ipdg_nodes(ipdg_ctx ctx, double* x, double* y, void* stream);

/* DG gradient and divergence with central fluxes (Eqs. INS_SD_4_1 / INS_SD_4_2):
 * the nodal operators G p = grad p + 1/2 sum_f (sJ/J) LIFT_f (n [[p]]) and D u = div u + 1/2 sum_f
 * (sJ/J) LIFT_f (n.[[u]]), i.e. (J^e M)^{-1} times the variational forms of the paper, used for the
 * pressure right-hand side -(gamma/dt) D.U and the velocity update U - (dt/gamma) G dP (Eq. INS_TD_3).
 * Homogeneous boundary data by mirroring, with the context's face codes read as PRESSURE types
 * (R20): IPDG_BC_DIRICHLET (outflow) p+ = -p-, u+ = u-; IPDG_BC_NEUMANN (velocity
 * Dirichlet) p+ = p-, u+ = -u-.  All fields K x Np device arrays, outputs distinct from inputs;
 * asynchronous on `stream`.  Single-partition contexts only (IPDG_ESTATE with a halo). */
int ipdg_dg_grad(ipdg_ctx ctx, const double* p, double* gx, double* gy, void* stream);
int ipdg_dg_div(ipdg_ctx ctx, const double* ux, const double* uy, double* d, void* stream);

/* Scratch for PCG: query the size, hand over caller-owned device memory (e.g. a torch
 * tensor).  Without ipdg_set_workspace the library allocates it itself on first use. */
int ipdg_workspace_bytes(ipdg_ctx ctx, int64_t* bytes);
int ipdg_set_workspace(ipdg_ctx ctx, void* dev, int64_t bytes);

/* Solve A x = b by PCG (R12), precond = IPDG_PRECOND_*: x in = x0, out = solution.
 * Stops when ||r_k||_2 <= tol ||b||_2 or after maxit iterations (IPDG_NOT_CONVERGED).
 * b = 0 returns x = 0 with 0 iterations.  Blocks until the result is known; the
 * iteration loop runs on the device (no host sync per iteration). */
int ipdg_pcg_solve(ipdg_ctx ctx, const double* b, double* x, double lambda, int precond, double tol,
                   int64_t maxit, ipdg_stats* stats, void* stream);

/* Split form used for timing fixed iteration windows (bench.py):
 *   begin:   r = b - A x, z = D^{-1} r, rho = r.z, ||b||   (async)
 *   iterate: exactly n more iterations unless converged/broken down (async; 2 fused
 *            kernels per iteration, launched as a captured CUDA graph)
 *   end:     final x update, copy stats to the host (blocks). */
int ipdg_pcg_begin(ipdg_ctx ctx, const double* b, double* x, double lambda, int precond, double tol,
                   void* stream);
int ipdg_pcg_iterate(ipdg_ctx ctx, int64_t n, void* stream);
int ipdg_pcg_end(ipdg_ctx ctx, ipdg_stats* stats, void* stream);
/* Like ipdg_pcg_iterate but launched kernel by kernel (no graph) with CUDA events around
 * each pass on `stream`; returns the summed device durations (ms) of pass A (fused
 * direction update + Ax + p.Ap) and pass B (residual update + dots).  Synchronizes. */
int ipdg_pcg_iterate_profiled(ipdg_ctx ctx, int64_t n, double* ms_pass_a, double* ms_pass_b, void* stream);

/* Subcycling advection operator (NEXT-4; Eq. INS_CUB_N, Eq. KSS_3, Alg. SSV / SSS):
 * (Nu, Nv) = N~(U_bar, U~) for the advective velocity (ub, vb) and the advected field (ut, vt), device
 * vectors K x Np each, nodal output (the (J M)^{-1} of the weak form applied).  Cubature exact to degree
 * 3N (volume: collapsed Gauss-Legendre; faces: Gauss-Legendre), local Lax-Friedrichs flux with
 * Lambda = max |n.U_bar+-| and Alg. SSS's dissipative sign (R27); boundary traces by the
 * velocity mirrors of the face codes (R28: code 1 U+ = U-, code 2 U+ = -U-).  One partition only. */
int ipdg_advect(ipdg_ctx ctx, const double* ub, const double* vb, const double* ut, const double* vt, double* Nu,
                double* Nv, void* stream);

/* One p-multigrid V-cycle z = B r (IPDG_PRECOND_PMG's preconditioner, R22-R26),
 * device vectors K x Np, builds the level hierarchy for `lambda` on first use (child contexts of
 * degrees N/2, ..., 1 on the same mesh, their diagonals and power-iteration lmax).  Async on `stream`
 * after the first (blocking) setup.  ipdg_pmg_info: number of levels (and, up to cap, their degrees
 * and lmax estimates) of the current hierarchy (0 before setup). */
int ipdg_pmg_apply(ipdg_ctx ctx, const double* r, double* z, double lambda, void* stream);
int ipdg_pmg_info(ipdg_ctx ctx, int* degrees, double* lmax, int cap);

/* Host-buffer convenience (the e2e path): copies b (host) in, solves, copies x out. */
int ipdg_pcg_solve_host(ipdg_ctx ctx, const double* b_host, double* x_host, double lambda, int precond,
                        double tol, int64_t maxit, ipdg_stats* stats, void* stream);

/* Every blocking call of the multi-GPU path waits by polling (cudaEventQuery) and checks
 * ncclCommGetAsyncError on each poll: a failed or hung peer aborts the communicator and returns
 * IPDG_ENCCL instead of blocking forever.  Timeout: environment IPDG_WAIT_TIMEOUT_S (default 600 s). */

/* ---- multi-GPU (one process per GPU; NCCL over NVLink) ----
 * ipdg_comm_init: nccl_unique_id points to the 128-byte ncclUniqueId broadcast by the caller
 * (e.g. through torch.distributed); call before ipdg_upload_mesh.  Faces coded
 * IPDG_BC_REMOTE are then matched across ranks through the global vertex ids in EToV
 * (same vertex numbering on every rank), and the PCG dot products are all-reduced. */
int ipdg_comm_init(ipdg_ctx ctx, const void* nccl_unique_id, int nranks, int rank);

/* Single-process loopback of the distributed PCG (tests; P:219 PCG with P:382 distribution):
 * cs[0..P-1] are contexts on ONE device holding the partitions of one mesh, each completed by
 * ipdg_upload_halo with neighbour ranks that index cs (no ipdg_comm_init).  b[p], x[p] are device
 * vectors of context p (K_p x Np; x[p] holds x0 on entry, the solution on return).  Every step of the
 * NCCL path runs in lockstep on `stream` -- p_k packing with pass A's decisions, halo exchange as
 * device-to-device copies in the plans' order, pass A (interior / halo-boundary launches and the
 * two-part p.Ap reduction), pass B -- and each NCCL all-reduce is a fixed-order sum over the P device
 * states.  stats[p] (optional, P entries) as ipdg_pcg_solve.  Returns as ipdg_pcg_solve; blocks. */
int ipdg_loopback_pcg_solve(ipdg_ctx* cs, int P, const double* const* b, double* const* x, double lambda,
                            int precond, double tol, int64_t maxit, ipdg_stats* stats, void* stream);

/* Complete a mesh uploaded with IPDG_BC_REMOTE faces (multi-GPU partition, built e.g. by
 * paper_1801_00246_b200.partition.split).  HOST arrays, copied:
 *   H              ghost elements owned by other ranks (local ids K .. K+H-1)
 *   ghost_etov     [H*3] their global vertex ids (coordinates from the VX, VY of ipdg_upload_mesh)
 *   remote         [K*3] ghost index h on IPDG_BC_REMOTE faces (else ignored)
 *   remote_face    [K*3] the ghost's face index f' on those faces
 *   nnbr, nbr_rank [nnbr] neighbour ranks; send_off/recv_off [nnbr+1] offsets;
 *   send_elem      [send_off[nnbr]] local element ids sent to each neighbour, in the order the
 *                  neighbour stores them as ghosts (its recv list from this rank).
 * Every ipdg_ax / PCG iteration then exchanges the ghost rows with NCCL send/recv on the
 * caller's stream before the operator kernel. */
int ipdg_upload_halo(ipdg_ctx ctx, int64_t H, const int32_t* ghost_etov, const int32_t* remote,
                     const int8_t* remote_face, int nnbr, const int32_t* nbr_rank, const int64_t* send_off,
                     const int32_t* send_elem, const int64_t* recv_off);
/* Halo introspection / single-process exchange (tests): S sent rows, H ghost rows; pack the
 * S x Np rows of a field in plan order; install H x Np ghost rows (disables the NCCL exchange). */
int ipdg_halo_info(ipdg_ctx ctx, int64_t* S, int64_t* H);
int ipdg_halo_pack(ipdg_ctx ctx, const double* u, double* out, void* stream);
int ipdg_halo_set(ipdg_ctx ctx, const double* in, void* stream);
int ipdg_nccl_id_bytes(void);
int ipdg_nccl_get_unique_id(void* out128);

/* ---- introspection / test hooks ---- */
#define IPDG_OP_R 0     /* Np        node r */
#define IPDG_OP_S 1     /* Np        node s */
#define IPDG_OP_DR 2    /* Np*Np     row-major */
#define IPDG_OP_DS 3    /* Np*Np */
#define IPDG_OP_M 4     /* Np*Np     reference mass */
#define IPDG_OP_M1D 5   /* Nfp*Nfp   1-D face mass */
#define IPDG_OP_LIFT 6  /* Np*3Nfp   LIFT = M^{-1} E */
#define IPDG_OP_FMASK 7 /* 3*Nfp     (as doubles) */
int ipdg_get_refop(ipdg_ctx ctx, int which, double* host, int64_t cap);
/* Same tables without a context or a GPU (host-only setup code; returns the count). */
int ipdg_refop_host(int N, int which, double* host, int64_t cap);
/* K*5 doubles per element: rx, sx, ry, sy, J */
int ipdg_get_geofacs(ipdg_ctx ctx, double* host, int64_t cap);
/* K*3 neighbour element (-1 boundary) and K*3 neighbour face */
int ipdg_get_connectivity(ipdg_ctx ctx, int32_t* etoe, int32_t* etof, int64_t cap);
/* out[0..n), n <= 11: N, Np, K, nblocks, E (own elements per block), Gmax, smem bytes/CTA and grid of
 * k_sipdg, then the pass-A kernel the context resolves to for lambda = 0 (1 k_sipdg, 2 k_grad + k_flux,
 * 3 k_tpe, 4 k_pipe, 5 k_gather) with its smem bytes/CTA and grid */
int ipdg_info(ipdg_ctx ctx, int64_t* out, int n);
/* Operator kernel variant: 0 auto (the variant measured fastest for the degree and pass: Ax 5 for N <= 3,
 * 4 for N = 4, 5, 2 for N >= 6; PCG pass A 5 for N = 1, 4 for N = 2..5, 2 for N >= 6), 1 fused single-kernel (k_sipdg, DMMA), 2 split gradient + flux kernels
 * (k_grad, k_flux, DMMA), 3 thread-per-element with block staging (k_tpe, DFMA with operators in
 * constant memory), 4 software-pipelined fused (k_pipe, DMMA, TMA-staged rows; falls back to 1 when an
 * operand is not 16-byte aligned or the block does not fit in shared memory), 5 gather (k_gather, one
 * thread per element reading its neighbours' rows from L1/L2, DFMA).  Variants 3 and 5 need N <= 4
 * (else IPDG_EINVAL).  Results agree to rounding.  Switching drops captured CG graphs. */
int ipdg_set_variant(ipdg_ctx ctx, int variant);
/* number of kernel launches this context has issued (evidence counter) */
int64_t ipdg_launch_count(ipdg_ctx ctx);

const char* ipdg_strerror(int code);
int ipdg_last_error(ipdg_ctx ctx, char* buf, int cap);

#ifdef __cplusplus
}
#endif
#endif /* IPDG_H */
