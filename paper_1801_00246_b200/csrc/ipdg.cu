// libipdg: C ABI (include/ipdg.h) over the sm_100a SIPDG kernels.
// Paper: arXiv:1801.00246 (P:n = PAPER.md line n).  Design: DESIGN.md.
//
// Host responsibilities (setup, once per mesh): reference operators (refops.cpp),
// face connectivity by vertex-pair matching, the element-block schedule with its
// ghost lists, DMMA fragment tables, geometric factors (on the device), the Jacobi
// diagonal.  Hot path (every call): k_sipdg (Ax, or PCG pass A fused with the
// direction update and p.Ap), k_pcg_b (residual update fused with r.z and r.r),
// all on the caller's stream; PCG iterations are replayed from captured CUDA graphs.
//
// PCG protocol (device-resident scalars, PcgState):
//   begin:  Ap = A x0;  r = b - Ap;  red_B = (r.z, r.r, b.b)       [+ allreduce(3)]
//   iter k: pass A (k_sipdg MODE_PCG_A): decide stop from red_B (rr_{k-1} <= tol^2 bb,
//             or k-1 = maxit); else beta = rho_{k-1}/rho_{k-2}; p_k = D^-1 r + beta p_{k-1}
//             (double-buffered); x += alpha_{k-1} p_{k-1} (deferred); Ap = A p_k;
//             red_A = p_k . Ap                                          [+ allreduce(1)]
//           pass B (k_pcg_b): alpha_k = rho_{k-1}/red_A (breakdown if <= 0);
//             r -= alpha_k Ap; red_B = (r.z, r.r); it = k               [+ allreduce(2)]
//   end:    pending x += alpha_k p_k if no stop was decided; stats to host.
#include "ctx.h"

#include <chrono>
#include <cstdlib>
#include <thread>
#include "sipdg_kernels.cuh"
#include "sipdg_split.cuh"
#include "sipdg_pipe.cuh"
#include "pmg.cuh"

#include <numeric>


#define IPDG_DECL_OPS(N_) const ImplOps* impl_ops_##N_();
IPDG_DECL_OPS(1) IPDG_DECL_OPS(2) IPDG_DECL_OPS(3) IPDG_DECL_OPS(4)
IPDG_DECL_OPS(5) IPDG_DECL_OPS(6) IPDG_DECL_OPS(7) IPDG_DECL_OPS(8)
const ImplOps* impl_ops(int N) {
  switch (N) {
    case 1: return impl_ops_1(); case 2: return impl_ops_2(); case 3: return impl_ops_3(); case 4: return impl_ops_4();
    case 5: return impl_ops_5(); case 6: return impl_ops_6(); case 7: return impl_ops_7(); default: return impl_ops_8();
  }
}


#define DISPATCH(N_, CALL)                          \
  do {                                              \
    if ((N_) < 1 || (N_) > 8) return IPDG_EDEGREE;  \
    return impl_ops(N_)->CALL;                      \
  } while (0)

static int e_of(int N) {
  switch (N) {
    case 1: return Tr<1>::E; case 2: return Tr<2>::E; case 3: return Tr<3>::E; case 4: return Tr<4>::E;
    case 5: return Tr<5>::E; case 6: return Tr<6>::E; case 7: return Tr<7>::E; default: return Tr<8>::E;
  }
}
static std::vector<double> tables_of(const RefOps& R) { return impl_ops(R.N)->build_tables(R); }
static std::vector<double> diagtab_of(const RefOps& R) { return impl_ops(R.N)->build_diagtab(R); }

// largest ghost count per block that keeps k_sipdg<N> (lambda variant) within the SM's
// opt-in shared memory at one CTA per SM
template <int N>
static int ghost_cap_n(int device) {
  using T = Tr<N>;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (optin <= 0) optin = 227 * 1024;
  const int fixed = SmemLayout::make<N>(0, true, true).total * 8 + 1024;  // + static smem
  const int per = (T::SU + T::SG + 2 + std::max(T::SXY, 2 * T::NP)) * 8;  // slot + ids (+ PCG staging aliasing w)
  int g = (optin - fixed) / per;
  g = g / 8 * 8;
  return std::max(8, std::min(g, 30000 - T::E));
}
static int ghost_cap(int N, int device) {
  switch (N) {
    case 1: return ghost_cap_n<1>(device); case 2: return ghost_cap_n<2>(device);
    case 3: return ghost_cap_n<3>(device); case 4: return ghost_cap_n<4>(device);
    case 5: return ghost_cap_n<5>(device); case 6: return ghost_cap_n<6>(device);
    case 7: return ghost_cap_n<7>(device); default: return ghost_cap_n<8>(device);
  }
}

static void free_ws(ipdg_ctx c);

// drops every mesh-sized buffer, including the PCG workspace binding (its layout depends on K + H)
static void free_pmg(ipdg_ctx c) {
  for (auto& L : c->pmg) {
    if (L.ctx) ipdg_destroy(L.ctx);
    if (L.buf) cudaFree(L.buf);
    if (L.I) cudaFree(L.I);
  }
  c->pmg.clear();
  c->pmg_lambda = -1.0;
}

static void free_mesh(ipdg_ctx c) {
  free_ws(c);
  free_pmg(c);
  if (c->hostio) cudaFree(c->hostio);
  c->hostio = nullptr;
  c->hostio_n = 0;
  void* ptrs[] = {c->geo, c->gG, c->gF, c->nbr, c->goff, c->gid, c->boff, c->etoe, c->bcode, c->vxy, c->nbg, c->W2,
                  c->nbt, c->gfoff_t, c->gface_t, c->tauF, c->blist_t, c->adv_tab};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  c->nbt = nullptr; c->gfoff_t = nullptr; c->gface_t = nullptr; c->tauF = nullptr; c->blist_t = nullptr;
  c->adv_tab = nullptr;
  c->nblocks_t = 0; c->gmax_t = 0;
  c->geo = nullptr; c->gG = nullptr; c->gF = nullptr; c->nbr = nullptr; c->goff = nullptr; c->gid = nullptr; c->boff = nullptr; c->etoe = nullptr;
  c->nbg = nullptr; c->W2 = nullptr;
  c->bcode = nullptr;
  c->vxy = nullptr;
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  c->gkey_x = nullptr;
  c->dinv_valid = false;
  if (c->send_idx) cudaFree(c->send_idx);
  if (c->sendbuf) cudaFree(c->sendbuf);
  if (c->halobuf) cudaFree(c->halobuf);
  c->send_idx = nullptr; c->sendbuf = nullptr; c->halobuf = nullptr;
  c->S = 0; c->H = 0; c->K = 0; c->halo_external = false;
}

static void free_ws(ipdg_ctx c) {
  if (c->ws_owned && c->ws) cudaFree(c->ws);
  c->ws = nullptr;
  c->ws_owned = false;
  c->ws_bytes = 0;
  c->r = c->pe = c->po = c->Ap = c->dinv = c->zb = nullptr;
  c->dinv_valid = false;
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  c->gkey_x = nullptr;
}

extern "C" {

const char* ipdg_strerror(int code) {
  switch (code) {
    case IPDG_OK: return "ok";
    case IPDG_NOT_CONVERGED: return "not converged (maxit reached)";
    case IPDG_EINVAL: return "invalid argument";
    case IPDG_EDEGREE: return "degree N out of range 1..8";
    case IPDG_EMESH: return "invalid mesh";
    case IPDG_EBREAKDOWN: return "PCG breakdown (p^T A p <= 0)";
    case IPDG_ESINGULAR: return "singular operator (lambda = 0 and no Dirichlet face)";
    case IPDG_ECUDA: return "CUDA error";
    case IPDG_ENCCL: return "NCCL error";
    case IPDG_ESTATE: return "invalid call order";
    default: return "unknown error";
  }
}

int ipdg_last_error(ipdg_ctx c, char* buf, int cap) {
  if (!c || !buf || cap <= 0) return IPDG_EINVAL;
  snprintf(buf, cap, "%s", c->err.c_str());
  return IPDG_OK;
}

int ipdg_create(ipdg_ctx* out, int N, int device) {
  if (!out) return IPDG_EINVAL;
  *out = nullptr;
  if (N < 1 || N > 8) return IPDG_EDEGREE;
  ipdg_ctx c = new ipdg_ctx_s();
  c->N = N;
  c->device = device;
  c->E = e_of(N);
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return IPDG_ECUDA;
  }
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  try {
    c->ref = build_refops(N);
  } catch (const std::exception& e) {
    delete c;
    return IPDG_ECUDA;
  }
  const RefOps& R = c->ref;
  // the kernels use the closed-form face-node indices of kernels.cuh (fmask_cf); check them
  for (int f = 0; f < 3; ++f)
    for (int k = 0; k <= N; ++k) {
      const int off = k * (N + 1) - k * (k - 1) / 2;
      const int cf = f == 0 ? k : (f == 1 ? off + N - k : off);
      if (R.Fmask[f * (N + 1) + k] != cf) {
        delete c;
        return IPDG_EDEGREE;
      }
    }
  int rc = IPDG_OK;
  std::vector<double> tab = tables_of(R), dtab = diagtab_of(R), rs(2 * R.Np);
  for (int i = 0; i < R.Np; ++i) { rs[i] = R.r[i]; rs[R.Np + i] = R.s[i]; }
  if ((rc = upload(c, &c->tables, tab.data(), tab.size())) || (rc = upload(c, &c->diagtab, dtab.data(), dtab.size())) ||
      (rc = upload(c, &c->rs, rs.data(), rs.size())) || (rc = upload(c, &c->Mref, R.M.data(), R.M.size()))) {
    delete c;
    return rc;
  }
  if ((rc = impl_ops(N)->upload_constants(c))) {
    delete c;
    return rc;
  }
  if (cudaMalloc(&c->st, sizeof(PcgState)) != cudaSuccess || cudaMallocHost(&c->st_host, sizeof(PcgState)) != cudaSuccess ||
      cudaMalloc(&c->counter, sizeof(unsigned int)) != cudaSuccess || cudaMemset(c->counter, 0, sizeof(unsigned int)) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return IPDG_ECUDA;
  }
  *out = c;
  return IPDG_OK;
}

int ipdg_destroy(ipdg_ctx c) {
  if (!c) return IPDG_EINVAL;
  cudaSetDevice(c->device);
  free_mesh(c);
  free_ws(c);
  void* ptrs[] = {c->tables, c->diagtab, c->rs, c->Mref, c->Minv, c->dgops, c->st, c->counter, c->partials};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->st_host) cudaFreeHost(c->st_host);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->blist) cudaFree(c->blist);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return IPDG_OK;
}

static int finalize_mesh(ipdg_ctx c, int64_t H, const double* ghost_vxy);

int ipdg_upload_mesh(ipdg_ctx c, int64_t K, int64_t Nv, const double* VX, const double* VY, const int32_t* EToV,
                     const int8_t* bc, double tau_scale) {
  if (!c) return IPDG_EINVAL;
  if (K <= 0 || Nv <= 0 || !VX || !VY || !EToV || !bc || !(tau_scale > 0.0))
    FAIL(c, IPDG_EINVAL, "upload_mesh: bad arguments");
  if (K > (int64_t)INT32_MAX / 3) FAIL(c, IPDG_EINVAL, "upload_mesh: K too large");
  CUDA_TRY(c, cudaSetDevice(c->device));
  free_mesh(c);
  const int E = c->E;
  // ---- connectivity by sorting vertex-pair keys
  std::vector<std::pair<uint64_t, int64_t>> keys((size_t)K * 3);
  for (int64_t e = 0; e < K; ++e)
    for (int f = 0; f < 3; ++f) {
      const int64_t a = EToV[e * 3 + f], b = EToV[e * 3 + (f + 1) % 3];
      if (a < 0 || b < 0 || a >= Nv || b >= Nv || a == b) FAIL(c, IPDG_EMESH, "element %lld has an invalid vertex id", (long long)e);
      if (bc[e * 3 + f] < 0 || bc[e * 3 + f] > 3) FAIL(c, IPDG_EINVAL, "element %lld face %d: bad boundary code", (long long)e, f);
      keys[e * 3 + f] = {(uint64_t)std::min(a, b) * (uint64_t)Nv + (uint64_t)std::max(a, b), e * 3 + f};
    }
  std::sort(keys.begin(), keys.end());
  std::vector<int> etoe(K * 3, -1), etof(K * 3, -1);
  for (size_t i = 0; i < keys.size();) {
    size_t j = i + 1;
    while (j < keys.size() && keys[j].first == keys[i].first) ++j;
    if (j - i > 2) FAIL(c, IPDG_EMESH, "non-manifold edge (face id %lld)", (long long)keys[i].second);
    if (j - i == 2) {
      const int64_t a = keys[i].second, b = keys[i + 1].second;
      etoe[a] = (int)(b / 3); etof[a] = (int)(b % 3);
      etoe[b] = (int)(a / 3); etof[b] = (int)(a % 3);
    }
    i = j;
  }
  bool dir = false;
  int64_t nremote = 0;
  for (int64_t i = 0; i < K * 3; ++i) {
    if (bc[i] == IPDG_BC_INTERIOR && etoe[i] < 0) FAIL(c, IPDG_EMESH, "interior face (%lld,%lld) has no neighbour", (long long)(i / 3), (long long)(i % 3));
    if (bc[i] != IPDG_BC_INTERIOR && etoe[i] >= 0) FAIL(c, IPDG_EMESH, "boundary-coded face (%lld,%lld) has a neighbour", (long long)(i / 3), (long long)(i % 3));
    if (bc[i] == IPDG_BC_DIRICHLET) dir = true;
    if (bc[i] == IPDG_BC_REMOTE) ++nremote;
  }
  c->has_dirichlet = dir;
  c->pend_K = K;
  c->pend_etoe = std::move(etoe);
  c->pend_etof = std::move(etof);
  c->pend_bc.assign(bc, bc + K * 3);
  c->pend_vxy.resize(K * 6);
  for (int64_t e = 0; e < K; ++e)
    for (int v = 0; v < 3; ++v) {
      c->pend_vxy[e * 6 + 2 * v] = VX[EToV[e * 3 + v]];
      c->pend_vxy[e * 6 + 2 * v + 1] = VY[EToV[e * 3 + v]];
    }
  c->pend_VX.assign(VX, VX + Nv);
  c->pend_VY.assign(VY, VY + Nv);
  c->pend_etov.assign(EToV, EToV + K * 3);
  c->tau_scale = tau_scale;
  c->tau_c = 0.5 * (c->N + 1) * (c->N + 2) * tau_scale;
  c->pend_remote = nremote;
  if (nremote > 0) return IPDG_OK;  // completed by ipdg_upload_halo
  return finalize_mesh(c, 0, nullptr);
}

// Block schedule, device arrays, geometric factors and launch configuration for the mesh
// stored by ipdg_upload_mesh plus H halo ghosts (ghost element g has local id K + g).
// Element-block schedule: contiguous ranges of at most E own elements whose distinct outside face
// neighbours (ghosts) fit the budget gcap.  Well-ordered meshes (Morton, RCB) never hit the cap,
// scattered orderings get shorter blocks instead of failing.  Halo ghosts (id >= K) are ordinary
// ghosts whose values come from the received halo buffer.  Slots: own e - e0, ghosts E + index.
struct Schedule {
  std::vector<int> boff, goff, gid;
  std::vector<short4> nbr;
  int gmax = 0;
};
static Schedule build_schedule(int64_t K, int E, int gcap, const std::vector<int>& etoe, const std::vector<int>& etof,
                               const int8_t* bc) {
  Schedule S;
  S.boff.assign(1, 0);
  S.goff.assign(1, 0);
  S.nbr.resize(K);
  std::vector<int> gl;
  int64_t e0 = 0;
  while (e0 < K) {
    gl.clear();
    int64_t e1 = e0;
    while (e1 < K && e1 - e0 < E) {
      for (int f = 0; f < 3; ++f) {
        const int n = etoe[e1 * 3 + f];
        if (n >= 0 && (n < e0 || n > e1)) gl.push_back(n);
      }
      std::sort(gl.begin(), gl.end());
      gl.erase(std::unique(gl.begin(), gl.end()), gl.end());
      // neighbours inside [e0, e1] are own elements: drop them from the ghost list
      gl.erase(std::remove_if(gl.begin(), gl.end(), [&](int n) { return n >= e0 && n <= e1; }), gl.end());
      if ((int)gl.size() > gcap && e1 > e0) {  // roll back this element
        gl.clear();
        for (int64_t e = e0; e < e1; ++e)
          for (int f = 0; f < 3; ++f) {
            const int n = etoe[e * 3 + f];
            if (n >= 0 && (n < e0 || n >= e1)) gl.push_back(n);
          }
        std::sort(gl.begin(), gl.end());
        gl.erase(std::unique(gl.begin(), gl.end()), gl.end());
        break;
      }
      ++e1;
    }
    S.gmax = std::max<int>(S.gmax, (int)gl.size());
    for (int64_t e = e0; e < e1; ++e) {
      short sl[3] = {0, 0, 0};
      int flags = 0;
      for (int f = 0; f < 3; ++f) {
        const int n = etoe[e * 3 + f];
        int slot = 0;
        if (n >= 0) {
          if (n >= e0 && n < e1) slot = (int)(n - e0);
          else slot = E + (int)(std::lower_bound(gl.begin(), gl.end(), n) - gl.begin());
        }
        sl[f] = (short)slot;
        const int fp = n >= 0 ? etof[e * 3 + f] : 0;
        const int code = (bc[e * 3 + f] == IPDG_BC_REMOTE) ? IPDG_BC_INTERIOR : bc[e * 3 + f];
        flags |= ((fp & 3) | ((code & 3) << 2)) << (4 * f);
      }
      S.nbr[e] = make_short4(sl[0], sl[1], sl[2], (short)flags);
    }
    S.gid.insert(S.gid.end(), gl.begin(), gl.end());
    S.goff.push_back((int)S.gid.size());
    S.boff.push_back((int)e1);
    e0 = e1;
  }
  return S;
}

// interior / halo-boundary block lists of the split pass A (a block is boundary when one of its ghosts
// is a halo ghost, id >= K); with force_split (tests) odd blocks count as boundary
static int build_block_lists(ipdg_ctx c, int64_t K, const std::vector<int>& boff, const std::vector<int>& goff,
                             const std::vector<int>& gid) {
  const int nb = (int)boff.size() - 1;
  std::vector<int> in, bd;
  bool any_halo = false;
  for (int b = 0; b < nb; ++b) {
    bool halo = false;
    for (int g = goff[b]; g < goff[b + 1]; ++g) halo |= gid[g] >= K;
    any_halo |= halo;
    if (c->force_split ? (b & 1) : halo) bd.push_back(b);
    else in.push_back(b);
  }
  c->nb_split[0] = (int)in.size();
  c->nb_split[1] = (int)bd.size();
  in.insert(in.end(), bd.begin(), bd.end());
  if (in.empty()) in.push_back(0);
  TRY(upload(c, &c->blist, in.data(), in.size()));
  c->split_a = any_halo || c->force_split != 0;
  return IPDG_OK;
}

// k_tpb schedule: blocks of E = tpb_e(N) consecutive elements (one thread each).  Per own face a slot: the
// neighbour's position in the block (own element), E + g for the block's g-th ghost face (neighbour
// outside the block, incl. halo ghosts >= K), or the element itself on a boundary face; flags as nbr.
// Ghost faces are listed per block as (neighbour << 2) | neighbour's face, sorted by that face so that
// the recomputation of their traces stays warp-convergent.  The split pass A lists (interior blocks,
// then blocks with a halo ghost face) follow build_block_lists.
static int build_tpb(ipdg_ctx c, int64_t K, const std::vector<int>& etoe, const std::vector<int>& etof, const int8_t* bc) {
  const int E = tpb_e(c->N);
  const int nb = (int)((K + E - 1) / E);
  std::vector<short4> nbt(K);
  std::vector<int> gfoff(1, 0), gface;
  std::vector<int> in, bd;
  int gmax = 0;
  std::vector<std::pair<int, int>> gl;  // (face', neighbour) of this block's ghost faces, own face order
  std::vector<int> own_ref;             // per ghost entry: own element * 3 + face
  for (int b = 0; b < nb; ++b) {
    const int64_t e0 = (int64_t)b * E, e1 = std::min<int64_t>(K, e0 + E);
    gl.clear();
    own_ref.clear();
    for (int64_t e = e0; e < e1; ++e)
      for (int f = 0; f < 3; ++f) {
        const int n = etoe[e * 3 + f];
        if (n >= 0 && (n < e0 || n >= e1)) {
          gl.push_back({etof[e * 3 + f], (int)own_ref.size()});
          own_ref.push_back((int)(e * 3 + f));
        }
      }
    std::stable_sort(gl.begin(), gl.end(), [](const std::pair<int, int>& x, const std::pair<int, int>& y) { return x.first < y.first; });
    std::vector<int> gslot(own_ref.size());
    bool halo = false;
    for (size_t g = 0; g < gl.size(); ++g) {
      const int ef = own_ref[gl[g].second];
      const int n = etoe[ef];
      halo |= n >= K;
      gface.push_back((n << 2) | gl[g].first);
      gslot[gl[g].second] = E + (int)g;
    }
    gmax = std::max(gmax, (int)gl.size());
    gfoff.push_back((int)gface.size());
    if (c->force_split ? (b & 1) : halo) bd.push_back(b);
    else in.push_back(b);
    size_t gi = 0;
    for (int64_t e = e0; e < e1; ++e) {
      short sl[3];
      int flags = 0;
      for (int f = 0; f < 3; ++f) {
        const int n = etoe[e * 3 + f];
        int slot = (int)(e - e0);
        if (n >= 0) slot = (n >= e0 && n < e1) ? (int)(n - e0) : gslot[gi++];
        sl[f] = (short)slot;
        const int fp = n >= 0 ? etof[e * 3 + f] : 0;
        const int code = (bc[e * 3 + f] == IPDG_BC_REMOTE) ? IPDG_BC_INTERIOR : bc[e * 3 + f];
        flags |= ((fp & 3) | ((code & 3) << 2)) << (4 * f);
      }
      nbt[e] = make_short4(sl[0], sl[1], sl[2], (short)flags);
    }
  }
  if (E + gmax > 32000 || (K + c->H) >= (1ll << 29)) FAIL(c, IPDG_EMESH, "k_tpb schedule: %d ghost faces in a block", gmax);
  c->nblocks_t = nb;
  c->gmax_t = gmax;
  c->nbt_split[0] = (int)in.size();
  c->nbt_split[1] = (int)bd.size();
  in.insert(in.end(), bd.begin(), bd.end());
  if (gface.empty()) gface.push_back(0);
  TRY(upload(c, &c->nbt, nbt.data(), nbt.size()));
  TRY(upload(c, &c->gfoff_t, gfoff.data(), gfoff.size()));
  TRY(upload(c, &c->gface_t, gface.data(), gface.size()));
  TRY(upload(c, &c->blist_t, in.data(), in.size()));
  return IPDG_OK;
}

__global__ void k_tauf(int64_t K, const double* __restrict__ gF, double* __restrict__ tauF) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < K * 3) tauF[i] = gF[(i / 3) * kGF + 3 * (i % 3) + 2];
}

// debug grid cap (ipdg_debug_grid_cap): clamp every persistent grid so that small test meshes run
// several element blocks per CTA (the prefetch / ring paths of the pipelined kernels)
static void apply_grid_cap(ipdg_ctx c) {
  const int cap = c->grid_cap;
  if (cap <= 0) return;
  for (auto& m : c->grid)
    for (int& g : m) g = std::min(g, cap);
  for (auto& m : c->grid_pipe)
    for (int& g : m) if (g > 0) g = std::min(g, cap);
  for (auto& m : c->grid_flux)
    for (int& g : m) g = std::min(g, cap);
  c->grid_grad = std::min(c->grid_grad, cap);
}

static int finalize_mesh(ipdg_ctx c, int64_t H, const double* ghost_vxy) {
  free_ws(c);  // the workspace layout depends on K + H
  const int64_t K = c->pend_K;
  const int E = c->E;
  std::vector<int>& etoe = c->pend_etoe;
  std::vector<int>& etof = c->pend_etof;
  const int8_t* bc = c->pend_bc.data();
  Schedule S = build_schedule(K, E, ghost_cap(c->N, c->device), etoe, etof, bc);
  std::vector<int>& boff = S.boff;
  std::vector<int>& goff = S.goff;
  std::vector<int>& gid = S.gid;
  std::vector<short4>& nbr = S.nbr;
  const int gmax = S.gmax;
  const int nb = (int)boff.size() - 1;
  if (E + gmax > 32000) FAIL(c, IPDG_EMESH, "element ordering too scattered (a block has %d ghosts)", gmax);
  c->K = K;
  c->H = H;
  c->nblocks = nb;
  c->gmax = gmax;
  std::vector<double> vxy(c->pend_vxy);
  if (H > 0) vxy.insert(vxy.end(), ghost_vxy, ghost_vxy + H * 6);
  std::vector<int8_t> bcv(bc, bc + K * 3);
  TRY(upload(c, &c->vxy, vxy.data(), vxy.size()));
  TRY(upload(c, &c->nbr, nbr.data(), nbr.size()));
  TRY(upload(c, &c->goff, goff.data(), goff.size()));
  TRY(upload(c, &c->gid, gid.data(), gid.size()));
  TRY(upload(c, &c->boff, boff.data(), boff.size()));
  TRY(build_block_lists(c, K, boff, goff, gid));
  TRY(upload(c, &c->etoe, etoe.data(), etoe.size()));
  TRY(upload(c, &c->bcode, bcv.data(), bcv.size()));
  c->etoe_h = etoe;
  c->etof_h = etof;
  {  // split variant: neighbour element ids (self on boundary faces) + the same face codes
    std::vector<int4> nbg(K);
    for (int64_t e = 0; e < K; ++e) {
      int id[3];
      for (int f = 0; f < 3; ++f) id[f] = etoe[e * 3 + f] >= 0 ? etoe[e * 3 + f] : (int)e;
      nbg[e] = make_int4(id[0], id[1], id[2], (int)(unsigned short)nbr[e].w);
    }
    TRY(upload(c, &c->nbg, nbg.data(), nbg.size()));
  }
  const int64_t KH = K + H;
  CUDA_TRY(c, cudaMalloc(&c->geo, KH * sizeof(double4)));
  unsigned long long* bad = nullptr;
  CUDA_TRY(c, cudaMalloc(&bad, sizeof(unsigned long long)));
  const unsigned long long none = ~0ull;
  CUDA_TRY(c, cudaMemcpy(bad, &none, sizeof(none), cudaMemcpyHostToDevice));
  k_geometry<<<(unsigned)((KH + 255) / 256), 256>>>(KH, c->vxy, c->geo, bad);
  c->launches++;
  unsigned long long badh = none;
  CUDA_TRY(c, cudaMemcpy(&badh, bad, sizeof(badh), cudaMemcpyDeviceToHost));
  cudaFree(bad);
  if (badh != none) FAIL(c, IPDG_EMESH, "element %llu has J <= 0 (vertices must be counter-clockwise)", badh);
  CUDA_TRY(c, cudaMalloc(&c->gG, KH * sizeof(double4)));
  CUDA_TRY(c, cudaMalloc(&c->gF, std::max<int64_t>(1, K) * kGF * sizeof(double)));
  k_geofacs<<<(unsigned)((KH + 255) / 256), 256>>>(K, KH, c->geo, c->etoe, c->bcode, c->tau_c, c->gG, c->gF);
  c->launches++;
  TRY(build_tpb(c, K, etoe, etof, bc));
  CUDA_TRY(c, cudaMalloc(&c->tauF, std::max<int64_t>(1, K) * 3 * sizeof(double)));
  k_tauf<<<(unsigned)((K * 3 + 255) / 256), 256>>>(K, c->gF, c->tauF);
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  TRY(impl_ops(c->N)->configure(c));
  apply_grid_cap(c);
  return IPDG_OK;
}

int ipdg_upload_halo(ipdg_ctx c, int64_t H, const int32_t* ghost_etov, const int32_t* remote, const int8_t* remote_face,
                     int nnbr, const int32_t* nbr_rank, const int64_t* send_off, const int32_t* send_elem,
                     const int64_t* recv_off) {
  if (!c || H < 0 || nnbr < 0 || (H > 0 && (!ghost_etov || !remote || !remote_face)) ||
      (nnbr > 0 && (!nbr_rank || !send_off || !send_elem || !recv_off)))
    FAIL(c, IPDG_EINVAL, "upload_halo: bad arguments");
  if (c->pend_K == 0 || c->pend_remote == 0) FAIL(c, IPDG_ESTATE, "upload_halo needs a mesh with IPDG_BC_REMOTE faces");
  const int64_t K = c->pend_K, Nv = (int64_t)c->pend_VX.size();
  if (recv_off[nnbr] != H) FAIL(c, IPDG_EINVAL, "upload_halo: receive offsets do not cover H ghosts");
  for (int64_t i = 0; i < K * 3; ++i) {
    if (c->pend_bc[i] != IPDG_BC_REMOTE) continue;
    const int h = remote[i], fp = remote_face[i];
    if (h < 0 || h >= H || fp < 0 || fp > 2) FAIL(c, IPDG_EMESH, "remote face %lld has no valid ghost", (long long)i);
    c->pend_etoe[i] = (int)(K + h);
    c->pend_etof[i] = fp;
  }
  std::vector<double> gv(H * 6);
  for (int64_t g = 0; g < H; ++g)
    for (int v = 0; v < 3; ++v) {
      const int64_t id = ghost_etov[g * 3 + v];
      if (id < 0 || id >= Nv) FAIL(c, IPDG_EMESH, "ghost %lld has an invalid vertex id", (long long)g);
      gv[g * 6 + 2 * v] = c->pend_VX[id];
      gv[g * 6 + 2 * v + 1] = c->pend_VY[id];
    }
  c->nbr_rank.assign(nbr_rank, nbr_rank + nnbr);
  c->send_off.assign(send_off, send_off + nnbr + 1);
  c->recv_off.assign(recv_off, recv_off + nnbr + 1);
  const int64_t S = nnbr ? send_off[nnbr] : 0;
  TRY(upload(c, &c->send_idx, send_elem, (size_t)S));
  c->S = S;
  if (c->sendbuf) cudaFree(c->sendbuf);
  if (c->halobuf) cudaFree(c->halobuf);
  c->sendbuf = c->halobuf = nullptr;
  CUDA_TRY(c, cudaMalloc(&c->sendbuf, std::max<int64_t>(1, S) * c->ref.Np * sizeof(double)));
  CUDA_TRY(c, cudaMalloc(&c->halobuf, std::max<int64_t>(1, H) * c->ref.Np * sizeof(double)));
  CUDA_TRY(c, cudaMemset(c->halobuf, 0, std::max<int64_t>(1, H) * c->ref.Np * sizeof(double)));
  // a Dirichlet face on any rank makes the operator non-singular
  if (c->comm && c->nranks > 1) {
    double* flag = nullptr;
    CUDA_TRY(c, cudaMalloc(&flag, sizeof(double)));
    const double v = c->has_dirichlet ? 1.0 : 0.0;
    CUDA_TRY(c, cudaMemcpy(flag, &v, sizeof(v), cudaMemcpyHostToDevice));
    NCCL_TRY(c, ncclAllReduce(flag, flag, 1, ncclFloat64, ncclSum, c->comm, 0));
    double g = 0.0;
    CUDA_TRY(c, cudaMemcpy(&g, flag, sizeof(g), cudaMemcpyDeviceToHost));
    cudaFree(flag);
    c->has_dirichlet_global = g > 0.0;
  } else {
    c->has_dirichlet_global = c->has_dirichlet;
  }
  return finalize_mesh(c, H, gv.data());
}

// ---- halo exchange (multi-GPU): pack the rows other ranks need, NCCL send/recv into the halo buffer
__global__ void k_pack_rows(int64_t S, int NP, const int* __restrict__ idx, const double* __restrict__ u,
                            double* __restrict__ out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= S * NP) return;
  const int64_t s = t / NP;
  const int i = (int)(t - s * NP);
  out[t] = u[(int64_t)idx[s] * NP + i];
}

// p_k = D^-1 r + beta p_{k-1} at the send rows, with the same decisions as pass A's prologue
__global__ void k_pack_p(int64_t S, int NP, const int* __restrict__ idx, const double* __restrict__ z,
                         const double* p_even, const double* p_odd, const PcgState* st, double* __restrict__ out) {
  if (st->stop_iter >= 0) return;
  const long long k = st->it + 1;
  const bool first = (k == 1);
  const double beta = first ? 0.0 : st->red_B[0] / st->rho_hist[(k - 2) & 3];
  const double* pold = (k & 1) ? p_even : p_odd;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= S * NP) return;
  const int64_t s = t / NP;
  const int i = (int)(t - s * NP);
  const int64_t g = (int64_t)idx[s] * NP + i;
  out[t] = first ? z[g] : z[g] + beta * pold[g];
}

static int halo_exchange(ipdg_ctx c, cudaStream_t s) {
  const int NP = c->ref.Np;
  NCCL_TRY(c, ncclGroupStart());
  for (size_t j = 0; j < c->nbr_rank.size(); ++j) {
    const int64_t so = c->send_off[j], sn = c->send_off[j + 1] - so;
    const int64_t ro = c->recv_off[j], rn = c->recv_off[j + 1] - ro;
    if (sn) NCCL_TRY(c, ncclSend(c->sendbuf + so * NP, sn * NP, ncclFloat64, c->nbr_rank[j], c->comm, s));
    if (rn) NCCL_TRY(c, ncclRecv(c->halobuf + ro * NP, rn * NP, ncclFloat64, c->nbr_rank[j], c->comm, s));
  }
  NCCL_TRY(c, ncclGroupEnd());
  return IPDG_OK;
}

static int halo_for_field(ipdg_ctx c, const double* u, cudaStream_t s) {
  if (c->H == 0 && c->S == 0) return IPDG_OK;
  if (c->halo_external) return IPDG_OK;  // test mode: the caller filled the halo buffer
  if (!c->comm) FAIL(c, IPDG_ESTATE, "mesh has remote faces but no communicator (ipdg_comm_init)");
  const int64_t n = c->S * c->ref.Np;
  if (n) {
    k_pack_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->S, c->ref.Np, c->send_idx, u, c->sendbuf);
    c->launches++;
  }
  return halo_exchange(c, s);
}

int ipdg_halo_info(ipdg_ctx c, int64_t* S, int64_t* H) {
  if (!c || !S || !H) return IPDG_EINVAL;
  *S = c->S;
  *H = c->H;
  return IPDG_OK;
}

int ipdg_halo_pack(ipdg_ctx c, const double* u, double* out, void* stream) {
  if (!c || !u || !out) return IPDG_EINVAL;
  const int64_t n = c->S * c->ref.Np;
  if (n) {
    k_pack_rows<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(c->S, c->ref.Np, c->send_idx, u, out);
    c->launches++;
  }
  CUDA_TRY(c, cudaGetLastError());
  return IPDG_OK;
}

int ipdg_halo_set(ipdg_ctx c, const double* in, void* stream) {
  if (!c || !in) return IPDG_EINVAL;
  if (c->H == 0) FAIL(c, IPDG_ESTATE, "no halo");
  CUDA_TRY(c, cudaMemcpyAsync(c->halobuf, in, c->H * c->ref.Np * sizeof(double), cudaMemcpyDeviceToDevice,
                              (cudaStream_t)stream));
  c->halo_external = true;
  return IPDG_OK;
}

int ipdg_ax(ipdg_ctx c, const double* u, double* Au, double lambda, void* stream) {
  if (!c || !u || !Au || u == Au || !(lambda >= 0.0)) return c ? (c->err = "ipdg_ax: bad arguments", IPDG_EINVAL) : IPDG_EINVAL;
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "ipdg_ax before ipdg_upload_mesh (or ipdg_upload_halo)");
  TRY(halo_for_field(c, u, (cudaStream_t)stream));
  DISPATCH(c->N, ax(c, u, Au, lambda, (cudaStream_t)stream));
}

static int dgop_check(ipdg_ctx c) {
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "DG gradient/divergence before ipdg_upload_mesh");
  if (c->H > 0 || c->S > 0) FAIL(c, IPDG_ESTATE, "DG gradient/divergence: partitioned meshes are not supported");
  if (!c->dgops) {
    std::vector<double> t(c->ref.Dr);
    t.insert(t.end(), c->ref.Ds.begin(), c->ref.Ds.end());
    t.insert(t.end(), c->ref.LIFT.begin(), c->ref.LIFT.end());
    TRY(upload(c, &c->dgops, t.data(), t.size()));
  }
  return IPDG_OK;
}

int ipdg_dg_grad(ipdg_ctx c, const double* p, double* gx, double* gy, void* stream) {
  if (!c || !p || !gx || !gy || gx == gy || p == gx || p == gy) return c ? (c->err = "ipdg_dg_grad: bad arguments", IPDG_EINVAL) : IPDG_EINVAL;
  TRY(dgop_check(c));
  DISPATCH(c->N, dgop(c, false, p, nullptr, gx, gy, (cudaStream_t)stream));
}

int ipdg_dg_div(ipdg_ctx c, const double* ux, const double* uy, double* d, void* stream) {
  if (!c || !ux || !uy || !d || d == ux || d == uy) return c ? (c->err = "ipdg_dg_div: bad arguments", IPDG_EINVAL) : IPDG_EINVAL;
  TRY(dgop_check(c));
  DISPATCH(c->N, dgop(c, true, ux, uy, d, nullptr, (cudaStream_t)stream));
}

int ipdg_diag(ipdg_ctx c, double* d, double lambda, void* stream) {
  if (!c || !d || !(lambda >= 0.0)) return IPDG_EINVAL;
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "ipdg_diag before ipdg_upload_mesh");
  DISPATCH(c->N, diag(c, d, lambda, (cudaStream_t)stream));
}

int ipdg_mass(ipdg_ctx c, const double* u, double* Mu, void* stream) {
  if (!c || !u || !Mu || u == Mu) return IPDG_EINVAL;
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "ipdg_mass before ipdg_upload_mesh");
  DISPATCH(c->N, mass(c, u, Mu, (cudaStream_t)stream));
}

int ipdg_nodes(ipdg_ctx c, double* x, double* y, void* stream) {
  if (!c || !x || !y) return IPDG_EINVAL;
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "ipdg_nodes before ipdg_upload_mesh");
  const int64_t n = c->K * c->ref.Np;
  k_nodes<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(c->K, c->ref.Np, c->vxy, c->rs, x, y);
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  return IPDG_OK;
}

int ipdg_workspace_bytes(ipdg_ctx c, int64_t* bytes) {
  if (!c || !bytes) return IPDG_EINVAL;
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "workspace size needs a mesh");
  const int64_t n = (c->K + c->H) * c->ref.Np;
  *bytes = 6 * ((n * 8 + 255) / 256 * 256);
  return IPDG_OK;
}

static int bind_ws(ipdg_ctx c) {
  const int64_t n = (c->K + c->H) * c->ref.Np;
  const int64_t seg = (n * 8 + 255) / 256 * 256;
  char* b = (char*)c->ws;
  c->r = (double*)(b);
  c->pe = (double*)(b + seg);
  c->po = (double*)(b + 2 * seg);
  c->Ap = (double*)(b + 3 * seg);
  c->dinv = (double*)(b + 4 * seg);
  c->zb = (double*)(b + 5 * seg);
  c->dinv_valid = false;
  return IPDG_OK;
}

int ipdg_set_workspace(ipdg_ctx c, void* dev, int64_t bytes) {
  if (!c || !dev) return IPDG_EINVAL;
  int64_t need = 0;
  TRY(ipdg_workspace_bytes(c, &need));
  if (bytes < need) FAIL(c, IPDG_EINVAL, "workspace too small: %lld < %lld", (long long)bytes, (long long)need);
  // always re-bind: the segment offsets depend on the current mesh (K + H)
  free_ws(c);
  c->ws = dev;
  c->ws_bytes = bytes;
  c->ws_owned = false;
  return bind_ws(c);
}

static int ensure_ws(ipdg_ctx c) {
  int64_t need = 0;
  TRY(ipdg_workspace_bytes(c, &need));
  if (c->ws && c->ws_bytes >= need) return IPDG_OK;
  free_ws(c);
  CUDA_TRY(c, cudaMalloc(&c->ws, need));
  c->ws_owned = true;
  c->ws_bytes = need;
  return bind_ws(c);
}

static int ensure_partials(ipdg_ctx c) {
  // one slot per CTA of the largest reducing grid (k_gather: one CTA per kGatherThreads elements)
  const int need = (int)std::max<int64_t>(std::max<int64_t>(std::max(4096, 4 * c->sms * 16), (c->K + kGatherThreads - 1) / kGatherThreads),
                                           c->nblocks_t);
  if (c->partials && c->partials_cap >= need) return IPDG_OK;
  if (c->partials) cudaFree(c->partials);
  CUDA_TRY(c, cudaMalloc(&c->partials, 3 * sizeof(double) * need));
  c->partials_cap = need;
  return IPDG_OK;
}

__global__ void k_recip(int64_t n, double* d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) d[i] = 1.0 / d[i];
}

static int allreduce(ipdg_ctx c, double* buf, int n, cudaStream_t s) {
  if (c->comm && c->nranks > 1) NCCL_TRY(c, ncclAllReduce(buf, buf, n, ncclFloat64, ncclSum, c->comm, s));
  return IPDG_OK;
}

static int vec_grid(ipdg_ctx c) { return c->grid_cap > 0 ? c->grid_cap : std::min(c->sms * 8, 4096); }

static int halo_for_p(ipdg_ctx c, cudaStream_t s) {
  if (c->H == 0 && c->S == 0) return IPDG_OK;
  if (!c->comm) FAIL(c, IPDG_ESTATE, "distributed PCG needs a communicator (ipdg_comm_init)");
  const int64_t n = c->S * c->ref.Np;
  if (n) {
    k_pack_p<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->S, c->ref.Np, c->send_idx, c->precond ? c->zb : c->r,
                                                         c->pe, c->po, c->st, c->sendbuf);
    c->launches++;
  }
  return halo_exchange(c, s);
}

static int pmg_apply(ipdg_ctx c, cudaStream_t s);
static int pass_b(ipdg_ctx c, cudaStream_t s) {
  if (c->precond == IPDG_PRECOND_BLOCK_JACOBI) DISPATCH(c->N, pass_b_bj(c, false, nullptr, s));
  k_pcg_b<<<vec_grid(c), 256, 0, s>>>(c->K * c->ref.Np, c->r, c->Ap, c->precond == IPDG_PRECOND_JACOBI ? c->dinv : nullptr,
                                        c->zb, c->st, c->partials, c->counter, c->xb ? c->x : nullptr, c->pe, c->po);
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  if (c->precond == IPDG_PRECOND_PMG) TRY(pmg_apply(c, s));
  return IPDG_OK;
}

static int resolved_pass_a(ipdg_ctx c) {
  const bool lam = c->lambda != 0.0;
  return impl_ops(c->N)->resolve(c, 1, lam, c->x);
}

static int one_iteration(ipdg_ctx c, cudaStream_t s) {
  const int kern = resolved_pass_a(c);
  if (c->split_a && (kern == 4 || kern == 6 || (kern == 2 && c->H > 0))) {
    // halo exchange of p_k on the comm stream, overlapping the interior blocks of pass A
    c->halo_ev_pending = false;
    if ((c->H > 0 || c->S > 0) && !c->halo_external) {
      CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
      CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
      TRY(halo_for_p(c, c->comm_stream));
      CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_stream));
      c->halo_ev_pending = true;
    }
    const int rc = [&]() -> int { DISPATCH(c->N, pass_a(c, s)); }();
    c->halo_ev_pending = false;
    TRY(rc);
  } else {
    TRY(halo_for_p(c, s));
    TRY([&]() -> int { DISPATCH(c->N, pass_a(c, s)); }());
  }
  TRY(allreduce(c, &c->st->red_A, 1, s));
  TRY(pass_b(c, s));
  TRY(allreduce(c, c->st->red_B, 2, s));
  return IPDG_OK;
}

static int capture(ipdg_ctx c, int iters, cudaGraphExec_t* out) {
  cudaGraph_t g = nullptr;
  CUDA_TRY(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = IPDG_OK;
  const int64_t l0 = c->launches;
  for (int i = 0; i < iters && rc == IPDG_OK; ++i) rc = one_iteration(c, c->cap_stream);
  c->launches_per_iter = (int)((c->launches - l0) / std::max(1, iters));  // kernels in one replayed iteration
  c->launches = l0;  // captured, not launched
  cudaError_t e = cudaStreamEndCapture(c->cap_stream, &g);
  if (rc != IPDG_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) FAIL(c, IPDG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) FAIL(c, IPDG_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  return IPDG_OK;
}

// ---- p-multigrid preconditioner (IPDG_PRECOND_PMG; pmg.cuh, oracle/pmg.py, R22-R26)
static int level_ax(ipdg_ctx c, int l, const double* u, double* Au, cudaStream_t s) {
  ipdg_ctx lc = l == 0 ? c : c->pmg[l].ctx;
  DISPATCH(lc->N, ax(lc, u, Au, c->pmg_lambda, s));
}

static double* lvec(ipdg_ctx c, int l, int which) {  // 0 dinv, 1 b, 2 x, 3 r, 4 d, 5 t, 6 y
  auto& L = c->pmg[l];
  if (l == 0 && which == 0) return c->dinv;
  return L.buf + which * L.seg;
}

// R24 / R26: `steps` Chebyshev steps from x = 0 for A x = b at level l over [a, 1.1 lmax] (smoother: 2 steps,
// a = lmax / 10; coarsest level: kPmgCoarseSteps, a = 1.1 lmax / kPmgCoarseRatio)
// With Ab the right-hand side is the residual b - Ab (stored in the level's r); with acc the last step also
// adds the result to acc (the V-cycle correction) and, with rdot, reduces rho = rdot . acc into the state.
static int cheb(ipdg_ctx c, int l, const double* b, double* x, cudaStream_t s, const double* Ab = nullptr,
                double* acc = nullptr, const double* rdot = nullptr) {
  auto& L = c->pmg[l];
  const bool coarse = (l + 1 == (int)c->pmg.size());
  const int steps = coarse ? kPmgCoarseSteps : 2;
  const int64_t n = c->K * L.Np;
  const double cc = 1.1 * L.lmax, a = coarse ? cc / kPmgCoarseRatio : L.lmax / 10.0;
  const double theta = 0.5 * (cc + a), delta = 0.5 * (cc - a), sigma = theta / delta;
  double* d = lvec(c, l, 4);
  double* t = lvec(c, l, 5);
  const int g = (int)std::min<int64_t>((n + 255) / 256, 4096);
  double* r = lvec(c, l, 3);
  k_cheb0<<<g, 256, 0, s>>>(n, b, Ab, r, lvec(c, l, 0), 1.0 / theta, x, d, c->pmg_gate);
  c->launches++;
  const double* bb = Ab ? r : b;
  double rho = 1.0 / sigma;
  for (int m = 1; m < steps; ++m) {
    const double rho_new = 1.0 / (2.0 * sigma - rho);
    const bool last = (m + 1 == steps);
    TRY(level_ax(c, l, x, t, s));
    k_cheb1<<<g, 256, 0, s>>>(n, bb, t, lvec(c, l, 0), rho_new * rho, 2.0 * rho_new / delta, x, d, last ? acc : nullptr,
                              last ? rdot : nullptr, c->st, c->partials, c->counter, c->pmg_gate);
    c->launches++;
    rho = rho_new;
  }
  CUDA_TRY(c, cudaGetLastError());
  return IPDG_OK;
}

// R25: x = V_l(b), zero initial guess.  The residuals are formed inside the restriction and the
// post-smoother's first step, the correction x += y inside its last step (with rdot: and rho = rdot . x).
// Returns in *dot_done whether rho was reduced (not on a one-level hierarchy).
static int vcycle(ipdg_ctx c, int l, const double* b, double* x, cudaStream_t s, const double* rdot = nullptr,
                  bool* dot_done = nullptr) {
  TRY(cheb(c, l, b, x, s));
  if (l + 1 == (int)c->pmg.size()) return IPDG_OK;
  auto& L = c->pmg[l];
  auto& C = c->pmg[l + 1];
  const int64_t n = c->K * L.Np, nc = c->K * C.Np;
  double* t = lvec(c, l, 5);
  double* y = lvec(c, l, 6);
  TRY(level_ax(c, l, x, t, s));
  k_restrict<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(c->K, L.Np, C.Np, L.I, b, t, lvec(c, l + 1, 1), c->pmg_gate);
  c->launches++;
  TRY(vcycle(c, l + 1, lvec(c, l + 1, 1), lvec(c, l + 1, 2), s));
  k_prolong<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->K, L.Np, C.Np, L.I, lvec(c, l + 1, 2), x, 1, c->pmg_gate);
  c->launches++;
  TRY(level_ax(c, l, x, t, s));
  TRY(cheb(c, l, b, y, s, t, x, rdot));
  if (dot_done) *dot_done = rdot != nullptr;
  CUDA_TRY(c, cudaGetLastError());
  return IPDG_OK;
}

static int host_dot(ipdg_ctx c, int64_t n, const double* u, const double* v, double* dev, cudaStream_t s, double* out) {
  k_dot<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(n, u, v, dev, nullptr, c->partials, c->counter);
  c->launches++;
  CUDA_TRY(c, cudaMemcpyAsync(out, dev, sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  return IPDG_OK;
}

// R22-R24: levels d_0 = N > d_1 > ... > 1 (child contexts on the same mesh), Jacobi diagonals, lmax by
// 20 power iterations, transfer matrices.  Level 0's diagonal is c->dinv (computed by pcg_setup).
static int pmg_setup(ipdg_ctx c, double lambda, cudaStream_t s) {
  if (!c->pmg.empty() && c->pmg_lambda == lambda) return IPDG_OK;
  if (c->H > 0 || c->S > 0) FAIL(c, IPDG_ESTATE, "p-multigrid preconditioner: one partition only");
  free_pmg(c);
  c->pmg_lambda = lambda;
  std::vector<int> deg{c->N};
  while (deg.back() > 1) deg.push_back(std::max(1, deg.back() / 2));
  const int64_t K = c->K, Nv = (int64_t)c->pend_VX.size();
  for (size_t l = 0; l < deg.size(); ++l) {
    ipdg_ctx_s::PmgLevel L;
    L.N = deg[l];
    L.Np = (L.N + 1) * (L.N + 2) / 2;
    L.seg = (K * L.Np + 31) / 32 * 32;
    if (l > 0) {
      TRY(ipdg_create(&L.ctx, L.N, c->device));
      c->pmg.push_back(L);  // owned from here on (free_pmg)
      const int rc = ipdg_upload_mesh(L.ctx, K, Nv, c->pend_VX.data(), c->pend_VY.data(), c->pend_etov.data(),
                                      c->pend_bc.data(), c->tau_scale);
      if (rc != IPDG_OK) FAIL(c, rc, "p-multigrid level %d: %s", L.N, L.ctx->err.c_str());
      L.ctx->variant = c->variant;
    } else {
      c->pmg.push_back(L);
    }
    auto& P = c->pmg.back();
    CUDA_TRY(c, cudaMalloc(&P.buf, 7 * P.seg * sizeof(double)));
    if (l > 0) {
      TRY([&]() -> int { DISPATCH(P.N, diag(P.ctx, P.buf, lambda, s)); }());
      k_recip<<<(unsigned)((K * P.Np + 255) / 256), 256, 0, s>>>(K * P.Np, P.buf);
      c->launches++;
    }
  }
  for (size_t l = 0; l + 1 < deg.size(); ++l) {
    const RefOps& F = (l == 0) ? c->ref : c->pmg[l].ctx->ref;
    const RefOps& Cr = c->pmg[l + 1].ctx->ref;
    const std::vector<double> I = interp_matrix(F, Cr);
    TRY(upload(c, &c->pmg[l].I, I.data(), I.size()));
  }
  // lmax of D^{-1} A per level (R24)
  double* dev = nullptr;
  CUDA_TRY(c, cudaMalloc(&dev, sizeof(double)));
  for (size_t l = 0; l < deg.size(); ++l) {
    const int64_t n = K * c->pmg[l].Np;
    double* v = lvec(c, (int)l, 1);
    double* w = lvec(c, (int)l, 2);
    double* t = lvec(c, (int)l, 5);
    const int g = (int)std::min<int64_t>((n + 255) / 256, 4096);
    k_pmg_start<<<g, 256, 0, s>>>(n, v);
    double lam = 0.0;
    for (int it = 0; it < 20; ++it) {
      TRY(level_ax(c, (int)l, v, t, s));
      k_scale<<<g, 256, 0, s>>>(n, lvec(c, (int)l, 0), t, w);
      double ww = 0.0, vv = 0.0;
      TRY(host_dot(c, n, w, w, dev, s, &ww));
      TRY(host_dot(c, n, v, v, dev, s, &vv));
      lam = std::sqrt(ww) / std::sqrt(vv);
      TRY(host_dot(c, n, w, w, dev, s, &ww));  // leaves w.w in dev for the normalisation
      k_normalize<<<g, 256, 0, s>>>(n, w, dev, v);
      c->launches += 2;
    }
    c->pmg[l].lmax = lam;
  }
  cudaFree(dev);
  CUDA_TRY(c, cudaGetLastError());
  return IPDG_OK;
}

// z = V(r) and rho = r.z -> st->red_B[0] (after the Jacobi-free pass B / init wrote z = r and the norms)
static int pmg_apply(ipdg_ctx c, cudaStream_t s) {
  c->pmg_gate = c->st;
  bool dot_done = false;
  TRY(vcycle(c, 0, c->r, c->zb, s, c->r, &dot_done));
  if (!dot_done) {  // one-level hierarchy (N = 1): rho = r.z here
    const int64_t n = c->K * c->ref.Np;
    k_dot<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(n, c->r, c->zb, nullptr, c->st, c->partials, c->counter);
    c->launches++;
  }
  CUDA_TRY(c, cudaGetLastError());
  return IPDG_OK;
}

// PCG setup shared by ipdg_pcg_begin and the loopback group solve: argument checks, workspace, Jacobi
// diagonal, device state (no Ax, no iteration graphs)
static int pcg_setup(ipdg_ctx c, const double* b, double* x, double lambda, int precond, double tol, bool dir,
                     cudaStream_t s) {
  if (!c || !b || !x || !(lambda >= 0.0) || !(tol >= 0.0) || precond < 0 || precond > 3) return IPDG_EINVAL;
  if (precond == IPDG_PRECOND_BLOCK_JACOBI && !(lambda > 0.0))
    FAIL(c, IPDG_EINVAL, "block-Jacobi (scaled inverse mass) preconditioning needs lambda > 0");
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "pcg before ipdg_upload_mesh");
  if (lambda == 0.0 && !dir) FAIL(c, IPDG_ESINGULAR, "lambda = 0 and no Dirichlet face");
  TRY(ensure_ws(c));
  TRY(ensure_partials(c));
  const int64_t n = c->K * c->ref.Np;
  if (precond == IPDG_PRECOND_BLOCK_JACOBI && !c->Minv) {
    TRY(upload(c, &c->Minv, c->ref.Minv.data(), c->ref.Minv.size()));
  }
  if ((precond == IPDG_PRECOND_JACOBI || precond == IPDG_PRECOND_PMG) && !(c->dinv_valid && c->dinv_lambda == lambda)) {
    TRY([&]() -> int { DISPATCH(c->N, diag(c, c->dinv, lambda, s)); }());
    k_recip<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, c->dinv);
    c->launches++;
    c->dinv_valid = true;
    c->dinv_lambda = lambda;
  }
  if (precond == IPDG_PRECOND_PMG) TRY(pmg_setup(c, lambda, s));
  c->x = x;
  c->lambda = lambda;
  c->precond = precond;
  {
    const int kern = impl_ops(c->N)->resolve(c, 1, lambda != 0.0, x);
#ifndef IPDG_TPB_XB
#define IPDG_TPB_XB 0  // experiment: k_tpb leaves x += alpha p to pass B
#endif
    c->xb = (kern == 4 && c->pipe_xb[lambda != 0.0]) || (kern == 6 && IPDG_TPB_XB);
    // the split pass A's W buffer, before any iteration is captured into a graph (the Ax of x0 may run
    // on another variant, e.g. k_pipe at N = 6, and no longer allocate it)
    if (kern == 2 && !c->W2)
      CUDA_TRY(c, cudaMalloc(&c->W2, std::max<int64_t>(1, c->K + c->H) * 2 * c->ref.Np * sizeof(double)));
  }
  PcgState h;
  std::memset(&h, 0, sizeof(h));
  h.tol2 = tol * tol;
  h.maxit = INT64_MAX / 4;
  h.stop_iter = -1;
  h.precond = precond;
  *c->st_host = h;
  CUDA_TRY(c, cudaMemcpyAsync(c->st, c->st_host, sizeof(PcgState), cudaMemcpyHostToDevice, s));
  return IPDG_OK;
}

// r = b - A x (A x already in c->Ap), z, partial (r.z, r.r, b.b) -> st->red_B (before the all-reduce)
static int pcg_init_residual(ipdg_ctx c, const double* b, cudaStream_t s) {
  if (c->precond == IPDG_PRECOND_BLOCK_JACOBI) DISPATCH(c->N, pass_b_bj(c, true, b, s));
  k_pcg_init<<<vec_grid(c), 256, 0, s>>>(c->K * c->ref.Np, b, c->Ap, c->r, c->precond == IPDG_PRECOND_JACOBI ? c->dinv : nullptr,
                                         c->zb, c->st, c->partials, c->counter);
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  if (c->precond == IPDG_PRECOND_PMG) TRY(pmg_apply(c, s));
  return IPDG_OK;
}

int ipdg_pcg_begin(ipdg_ctx c, const double* b, double* x, double lambda, int precond, double tol, void* stream) {
  if (!c) return IPDG_EINVAL;
  const bool dir = (c->H > 0 || c->S > 0) ? c->has_dirichlet_global : c->has_dirichlet;
  cudaStream_t s = (cudaStream_t)stream;
  TRY(pcg_setup(c, b, x, lambda, precond, tol, dir, s));
  TRY(ipdg_ax(c, x, c->Ap, lambda, stream));
  TRY(pcg_init_residual(c, b, s));
  TRY(allreduce(c, c->st->red_B, 3, s));
  // (re)capture the iteration graphs when the operands changed
  if (c->gkey_x != (const void*)x || c->gkey_lambda != lambda || c->gkey_precond != precond || !c->gexec[0]) {
    for (auto& g : c->gexec)
      if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    TRY(capture(c, 1, &c->gexec[0]));
    TRY(capture(c, kChunk, &c->gexec[1]));
    c->gkey_x = x;
    c->gkey_lambda = lambda;
    c->gkey_precond = precond;
  }
  return IPDG_OK;
}

static int set_maxit(ipdg_ctx c, int64_t maxit, cudaStream_t s) {
  c->st_host->maxit = maxit;
  CUDA_TRY(c, cudaMemcpyAsync(&c->st->maxit, &c->st_host->maxit, sizeof(long long), cudaMemcpyHostToDevice, s));
  return IPDG_OK;
}

int ipdg_pcg_iterate(ipdg_ctx c, int64_t n, void* stream) {
  if (!c || n < 0) return IPDG_EINVAL;
  if (!c->gexec[0]) FAIL(c, IPDG_ESTATE, "ipdg_pcg_iterate before ipdg_pcg_begin");
  cudaStream_t s = (cudaStream_t)stream;
  while (n >= kChunk) {
    CUDA_TRY(c, cudaGraphLaunch(c->gexec[1], s));
    c->launches += (int64_t)c->launches_per_iter * kChunk;
    n -= kChunk;
  }
  while (n-- > 0) {
    CUDA_TRY(c, cudaGraphLaunch(c->gexec[0], s));
    c->launches += c->launches_per_iter;
  }
  return IPDG_OK;
}

int ipdg_pcg_iterate_profiled(ipdg_ctx c, int64_t n, double* ms_a, double* ms_b, void* stream) {
  if (!c || n < 0 || !ms_a || !ms_b) return IPDG_EINVAL;
  if (!c->gexec[0]) FAIL(c, IPDG_ESTATE, "ipdg_pcg_iterate_profiled before ipdg_pcg_begin");
  cudaStream_t s = (cudaStream_t)stream;
  constexpr int B = 64;
  cudaEvent_t ev[3 * B];
  for (auto& e : ev) CUDA_TRY(c, cudaEventCreate(&e));
  double ta = 0.0, tb = 0.0;
  int rc = IPDG_OK;
  while (n > 0 && rc == IPDG_OK) {
    const int m = (int)std::min<int64_t>(n, B);
    for (int i = 0; i < m && rc == IPDG_OK; ++i) {
      cudaEventRecord(ev[3 * i], s);
      if ((rc = halo_for_p(c, s)) != IPDG_OK) break;
      rc = [&]() -> int { DISPATCH(c->N, pass_a(c, s)); }();
      if (rc != IPDG_OK) break;
      if ((rc = allreduce(c, &c->st->red_A, 1, s)) != IPDG_OK) break;
      cudaEventRecord(ev[3 * i + 1], s);
      if ((rc = pass_b(c, s)) != IPDG_OK) break;
      cudaEventRecord(ev[3 * i + 2], s);
      if ((rc = allreduce(c, c->st->red_B, 2, s)) != IPDG_OK) break;
    }
    if (rc != IPDG_OK) break;
    if (cudaStreamSynchronize(s) != cudaSuccess) { rc = IPDG_ECUDA; break; }
    for (int i = 0; i < m; ++i) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]);
      cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]);
      ta += a;
      tb += b;
    }
    n -= m;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc != IPDG_OK) return rc;
  CUDA_TRY(c, cudaGetLastError());
  *ms_a = ta;
  *ms_b = tb;
  return IPDG_OK;
}

// Wait for `s` by polling: with a communicator, every poll also checks ncclCommGetAsyncError, and a
// failure or the timeout (IPDG_WAIT_TIMEOUT_S, default 600 s) aborts the communicator and fails with
// IPDG_ENCCL instead of blocking forever on a dead peer (failure detection).
static int wait_stream(ipdg_ctx c, cudaStream_t s) {
  if (!c->comm) {
    CUDA_TRY(c, cudaStreamSynchronize(s));
    return IPDG_OK;
  }
  static const double timeout = [] {
    const char* e = std::getenv("IPDG_WAIT_TIMEOUT_S");
    const double v = e ? std::atof(e) : 0.0;
    return v > 0.0 ? v : 600.0;
  }();
  cudaEvent_t ev;
  CUDA_TRY(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(c, cudaEventRecord(ev, s));
  const auto t0 = std::chrono::steady_clock::now();
  int rc = IPDG_OK;
  for (;;) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      c->err = std::string("wait: ") + cudaGetErrorString(q);
      rc = IPDG_ECUDA;
      break;
    }
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(c->comm, &ar) != ncclSuccess || ar != ncclSuccess) {
      c->err = std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar);
      rc = IPDG_ENCCL;
    } else if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout) {
      c->err = "NCCL wait timed out (IPDG_WAIT_TIMEOUT_S)";
      rc = IPDG_ENCCL;
    }
    if (rc != IPDG_OK) {
      ncclCommAbort(c->comm);  // unblocks the stream's NCCL kernels
      c->comm = nullptr;
      break;
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  cudaEventDestroy(ev);
  return rc;
}

int ipdg_pcg_end(ipdg_ctx c, ipdg_stats* stats, void* stream) {
  if (!c) return IPDG_EINVAL;
  if (!c->x) FAIL(c, IPDG_ESTATE, "ipdg_pcg_end before ipdg_pcg_begin");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = c->K * c->ref.Np;
  if (!c->xb) {
    k_pcg_final_x<<<vec_grid(c), 256, 0, s>>>(n, c->x, c->pe, c->po, c->st);
    c->launches++;
  }
  k_pcg_final_state<<<1, 1, 0, s>>>(c->st);
  c->launches++;
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaMemcpyAsync(c->st_host, c->st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  TRY(wait_stream(c, s));
  const PcgState& h = *c->st_host;
  if (stats) {
    stats->iterations = h.stop_iter;
    stats->bnorm = std::sqrt(h.bb);
    stats->rel_residual = h.bb > 0 ? std::sqrt(h.final_rr / h.bb) : 0.0;
    stats->status = h.status;
    stats->reserved = 0;
    stats->seconds = 0.0;
  }
  if (h.status == -4) FAIL(c, IPDG_EBREAKDOWN, "PCG breakdown at iteration %lld", (long long)h.stop_iter);
  return h.status == 1 ? IPDG_NOT_CONVERGED : IPDG_OK;
}

int ipdg_pcg_solve(ipdg_ctx c, const double* b, double* x, double lambda, int precond, double tol, int64_t maxit,
                   ipdg_stats* stats, void* stream) {
  if (!c || maxit < 0) return IPDG_EINVAL;
  const auto t_start = std::chrono::steady_clock::now();
  cudaStream_t s = (cudaStream_t)stream;
  TRY(ipdg_pcg_begin(c, b, x, lambda, precond, tol, stream));
  TRY(set_maxit(c, maxit, s));
  int64_t done = 0;
  int64_t chunk = (precond == IPDG_PRECOND_PMG) ? 4 : kChunk;
  while (true) {
    const int64_t n = std::min<int64_t>(chunk, maxit + 1 - done);
    if (n <= 0) break;
    TRY(ipdg_pcg_iterate(c, n, stream));
    done += n;
    CUDA_TRY(c, cudaMemcpyAsync(&c->st_host->stop_iter, &c->st->stop_iter, sizeof(long long), cudaMemcpyDeviceToHost, s));
    TRY(wait_stream(c, s));
    if (c->st_host->stop_iter >= 0) break;
    // a p-multigrid iteration is ~10 Ax: short chunks (the level Ax kernels are not gated by the stop)
    chunk = (precond == IPDG_PRECOND_PMG) ? 4 : std::min<int64_t>(chunk * 2, 8 * kChunk);
  }
  const int rc = ipdg_pcg_end(c, stats, stream);
  if (stats) stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return rc;
}

int ipdg_pcg_solve_host(ipdg_ctx c, const double* b_host, double* x_host, double lambda, int precond, double tol,
                        int64_t maxit, ipdg_stats* stats, void* stream) {
  if (!c || !b_host || !x_host) return IPDG_EINVAL;
  const auto t_start = std::chrono::steady_clock::now();
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "pcg before ipdg_upload_mesh");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(ensure_ws(c));
  const int64_t n = c->K * c->ref.Np;
  // per-context device staging of b and x on the context's device, each vector 256-byte aligned (the
  // pipelined kernels move rows with bulk copies); allocated once per mesh, freed with it, so repeated
  // calls reuse the same pointers and the captured iteration graphs
  const int64_t seg = (n * 8 + 255) / 256 * 256 / 8;
  CUDA_TRY(c, cudaSetDevice(c->device));
  if (c->hostio_n < seg) {
    if (c->hostio) cudaFree(c->hostio);
    c->hostio = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->hostio, 2 * seg * sizeof(double)));
    c->hostio_n = seg;
  }
  double* bd = c->hostio;
  double* xd = c->hostio + c->hostio_n;
  CUDA_TRY(c, cudaMemcpyAsync(bd, b_host, n * sizeof(double), cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(xd, x_host, n * sizeof(double), cudaMemcpyHostToDevice, s));
  const int rc = ipdg_pcg_solve(c, bd, xd, lambda, precond, tol, maxit, stats, stream);
  if (rc < 0) return rc;
  CUDA_TRY(c, cudaMemcpyAsync(x_host, xd, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  TRY(wait_stream(c, s));
  if (stats) stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return rc;
}

// ---- single-process loopback of the distributed PCG (tests; SURVEY T4'): P contexts on one device hold
// the partitions of one mesh (ipdg_upload_halo plans whose neighbour ranks index `cs`).  The driver runs
// every step of the NCCL path in lockstep on one stream -- p_k packing with pass A's decisions (k_pack_p),
// the halo exchange (device-to-device copies from each sender's send buffer into the receivers' halo
// buffers, in the plans' order), pass A (interior / halo-boundary launches with the two-part p.Ap
// reduction when the halo split is active), pass B -- and replaces each NCCL all-reduce by a fixed-order
// sum over the P device states.
__global__ void k_group_sum(PcgState* const* sts, int P, int which, int n) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int j = 0; j < n; ++j) {
    double v = 0.0;
    for (int p = 0; p < P; ++p) v += (which == 0 ? &sts[p]->red_A : sts[p]->red_B)[j];
    for (int p = 0; p < P; ++p) (which == 0 ? &sts[p]->red_A : sts[p]->red_B)[j] = v;
  }
}

static int loop_exchange(ipdg_ctx* cs, int P, cudaStream_t s) {
  for (int r = 0; r < P; ++r) {
    ipdg_ctx c = cs[r];
    const int NP = c->ref.Np;
    for (size_t j = 0; j < c->nbr_rank.size(); ++j) {
      const int q = c->nbr_rank[j];
      if (q < 0 || q >= P || q == r) FAIL(c, IPDG_EINVAL, "loopback: neighbour rank %d outside the group", q);
      ipdg_ctx src = cs[q];
      size_t jj = 0;
      while (jj < src->nbr_rank.size() && src->nbr_rank[jj] != r) ++jj;
      if (jj == src->nbr_rank.size()) FAIL(c, IPDG_EMESH, "loopback: rank %d does not list rank %d", q, r);
      const int64_t n = src->send_off[jj + 1] - src->send_off[jj], rn = c->recv_off[j + 1] - c->recv_off[j];
      if (n != rn) FAIL(c, IPDG_EMESH, "loopback: rank %d sends %lld rows, rank %d expects %lld", q, (long long)n, r, (long long)rn);
      if (n)
        CUDA_TRY(c, cudaMemcpyAsync(c->halobuf + c->recv_off[j] * NP, src->sendbuf + src->send_off[jj] * NP,
                                    n * NP * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }
  return IPDG_OK;
}

int ipdg_loopback_pcg_solve(ipdg_ctx* cs, int P, const double* const* b, double* const* x, double lambda, int precond,
                            double tol, int64_t maxit, ipdg_stats* stats, void* stream) {
  if (!cs || P < 1 || !b || !x || maxit < 0) return IPDG_EINVAL;
  const auto t_start = std::chrono::steady_clock::now();
  for (int p = 0; p < P; ++p)
    if (!cs[p] || cs[p]->N != cs[0]->N || cs[p]->device != cs[0]->device || !b[p] || !x[p]) return IPDG_EINVAL;
  if (precond == IPDG_PRECOND_PMG) FAIL(cs[0], IPDG_ESTATE, "loopback PCG: p-multigrid needs one partition");
  cudaStream_t s = (cudaStream_t)stream;
  bool dir = false;
  for (int p = 0; p < P; ++p) dir |= cs[p]->has_dirichlet;
  for (int p = 0; p < P; ++p) {
    ipdg_ctx c = cs[p];
    CUDA_TRY(c, cudaSetDevice(c->device));
    c->has_dirichlet_global = dir;
    TRY(pcg_setup(c, b[p], x[p], lambda, precond, tol, dir, s));
    c->halo_ev_pending = false;
  }
  PcgState** dsts = nullptr;
  {
    std::vector<PcgState*> h(P);
    for (int p = 0; p < P; ++p) h[p] = cs[p]->st;
    CUDA_TRY(cs[0], cudaMalloc(&dsts, P * sizeof(PcgState*)));
    CUDA_TRY(cs[0], cudaMemcpy(dsts, h.data(), P * sizeof(PcgState*), cudaMemcpyHostToDevice));
  }
  auto run = [&]() -> int {
    // r = b - A x0 with x0's halo
    for (int p = 0; p < P; ++p) {
      ipdg_ctx c = cs[p];
      const int64_t n = c->S * c->ref.Np;
      if (n) {
        k_pack_rows<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->S, c->ref.Np, c->send_idx, x[p], c->sendbuf);
        c->launches++;
      }
    }
    TRY(loop_exchange(cs, P, s));
    for (int p = 0; p < P; ++p) {
      ipdg_ctx c = cs[p];
      TRY([&]() -> int { DISPATCH(c->N, ax(c, x[p], c->Ap, lambda, s)); }());
      TRY(pcg_init_residual(c, b[p], s));
    }
    k_group_sum<<<1, 1, 0, s>>>(dsts, P, 1, 3);
    for (int p = 0; p < P; ++p) TRY(set_maxit(cs[p], maxit, s));
    int64_t done = 0;
    while (done <= maxit) {
      const int64_t chunk = std::min<int64_t>(kChunk, maxit + 1 - done);
      for (int64_t it = 0; it < chunk; ++it) {
        for (int p = 0; p < P; ++p) {
          ipdg_ctx c = cs[p];
          const int64_t n = c->S * c->ref.Np;
          if (n) {
            k_pack_p<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c->S, c->ref.Np, c->send_idx, c->precond ? c->zb : c->r,
                                                                 c->pe, c->po, c->st, c->sendbuf);
            c->launches++;
          }
        }
        TRY(loop_exchange(cs, P, s));
        for (int p = 0; p < P; ++p) TRY([&]() -> int { DISPATCH(cs[p]->N, pass_a(cs[p], s)); }());
        k_group_sum<<<1, 1, 0, s>>>(dsts, P, 0, 1);
        for (int p = 0; p < P; ++p) TRY(pass_b(cs[p], s));
        k_group_sum<<<1, 1, 0, s>>>(dsts, P, 1, 2);
        CUDA_TRY(cs[0], cudaGetLastError());
      }
      done += chunk;
      ipdg_ctx c0 = cs[0];
      CUDA_TRY(c0, cudaMemcpyAsync(&c0->st_host->stop_iter, &c0->st->stop_iter, sizeof(long long), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(c0, cudaStreamSynchronize(s));
      if (c0->st_host->stop_iter >= 0) break;
    }
    for (int p = 0; p < P; ++p) {
      const int rc = ipdg_pcg_end(cs[p], stats ? &stats[p] : nullptr, stream);
      if (rc < 0) return rc;
      if (p == P - 1) return rc;
    }
    return IPDG_OK;
  };
  const int rc = run();
  cudaFree(dsts);
  if (stats)
    for (int p = 0; p < P; ++p) stats[p].seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return rc;
}

int ipdg_advect(ipdg_ctx c, const double* ub, const double* vb, const double* ut, const double* vt, double* Nu, double* Nv,
                void* stream) {
  if (!c || !ub || !vb || !ut || !vt || !Nu || !Nv || Nu == Nv) return IPDG_EINVAL;
  for (const double* in : {ub, vb, ut, vt})
    if (in == Nu || in == Nv) FAIL(c, IPDG_EINVAL, "ipdg_advect: outputs must not alias the inputs");
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "ipdg_advect before ipdg_upload_mesh");
  if (c->H > 0 || c->S > 0) FAIL(c, IPDG_ESTATE, "ipdg_advect: partitioned meshes are not supported");
  const double* f[4] = {ub, vb, ut, vt};
  double* o[2] = {Nu, Nv};
  DISPATCH(c->N, advect(c, f, o, (cudaStream_t)stream));
}

int ipdg_pmg_apply(ipdg_ctx c, const double* r, double* z, double lambda, void* stream) {
  if (!c || !r || !z || r == z || !(lambda >= 0.0)) return IPDG_EINVAL;
  if (c->K == 0) FAIL(c, IPDG_ESTATE, "ipdg_pmg_apply before ipdg_upload_mesh");
  cudaStream_t s = (cudaStream_t)stream;
  TRY(ensure_ws(c));
  TRY(ensure_partials(c));
  const int64_t n = c->K * c->ref.Np;
  if (!(c->dinv_valid && c->dinv_lambda == lambda)) {
    TRY([&]() -> int { DISPATCH(c->N, diag(c, c->dinv, lambda, s)); }());
    k_recip<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, c->dinv);
    c->launches++;
    c->dinv_valid = true;
    c->dinv_lambda = lambda;
  }
  TRY(pmg_setup(c, lambda, s));
  c->pmg_gate = nullptr;
  return vcycle(c, 0, r, z, s);
}

int ipdg_pmg_info(ipdg_ctx c, int* degrees, double* lmax, int cap) {
  if (!c || cap < 0) return IPDG_EINVAL;
  const int L = (int)c->pmg.size();
  for (int l = 0; l < L && l < cap; ++l) {
    if (degrees) degrees[l] = c->pmg[l].N;
    if (lmax) lmax[l] = c->pmg[l].lmax;
  }
  return L;
}

int ipdg_comm_init(ipdg_ctx c, const void* id, int nranks, int rank) {
  if (!c || !id || nranks < 1 || rank < 0 || rank >= nranks) return IPDG_EINVAL;
  CUDA_TRY(c, cudaSetDevice(c->device));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  if (c->comm) ncclCommDestroy(c->comm);
  NCCL_TRY(c, ncclCommInitRank(&c->comm, nranks, uid, rank));
  c->nranks = nranks;
  c->rank = rank;
  return IPDG_OK;
}

int ipdg_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int ipdg_nccl_get_unique_id(void* out) {
  if (!out) return IPDG_EINVAL;
  ncclUniqueId uid;
  if (ncclGetUniqueId(&uid) != ncclSuccess) return IPDG_ENCCL;
  std::memcpy(out, &uid, sizeof(uid));
  return IPDG_OK;
}

static int refop_copy(const RefOps& R, int which, double* host, int64_t cap);
int ipdg_get_refop(ipdg_ctx c, int which, double* host, int64_t cap) {
  if (!c || !host) return IPDG_EINVAL;
  return refop_copy(c->ref, which, host, cap);
}

int ipdg_refop_host(int N, int which, double* host, int64_t cap) {
  if (!host) return IPDG_EINVAL;
  if (N < 1 || N > 8) return IPDG_EDEGREE;
  try {
    return refop_copy(build_refops(N), which, host, cap);
  } catch (const std::exception&) {
    return IPDG_EINVAL;
  }
}

static int refop_copy(const RefOps& R, int which, double* host, int64_t cap) {
  std::vector<double> v;
  switch (which) {
    case IPDG_OP_R: v = R.r; break;
    case IPDG_OP_S: v = R.s; break;
    case IPDG_OP_DR: v = R.Dr; break;
    case IPDG_OP_DS: v = R.Ds; break;
    case IPDG_OP_M: v = R.M; break;
    case IPDG_OP_M1D: v = R.M1D; break;
    case IPDG_OP_LIFT: v = R.LIFT; break;
    case IPDG_OP_FMASK: v.assign(R.Fmask.begin(), R.Fmask.end()); break;
    default: return IPDG_EINVAL;
  }
  if (cap < (int64_t)v.size()) return IPDG_EINVAL;
  std::copy(v.begin(), v.end(), host);
  return (int)v.size();
}

int ipdg_get_geofacs(ipdg_ctx c, double* host, int64_t cap) {
  if (!c || !host) return IPDG_EINVAL;
  if (c->K == 0) return IPDG_ESTATE;
  if (cap < c->K * 5) return IPDG_EINVAL;
  std::vector<double4> g(c->K);
  CUDA_TRY(c, cudaMemcpy(g.data(), c->geo, c->K * sizeof(double4), cudaMemcpyDeviceToHost));
  for (int64_t e = 0; e < c->K; ++e) {
    host[e * 5 + 0] = g[e].x; host[e * 5 + 1] = g[e].y; host[e * 5 + 2] = g[e].z; host[e * 5 + 3] = g[e].w;
    host[e * 5 + 4] = 1.0 / (g[e].x * g[e].w - g[e].y * g[e].z);
  }
  return IPDG_OK;
}

int ipdg_get_connectivity(ipdg_ctx c, int32_t* etoe, int32_t* etof, int64_t cap) {
  if (!c || !etoe || !etof) return IPDG_EINVAL;
  if (c->K == 0) return IPDG_ESTATE;
  if (cap < c->K * 3) return IPDG_EINVAL;
  std::copy(c->etoe_h.begin(), c->etoe_h.end(), etoe);
  std::copy(c->etof_h.begin(), c->etof_h.end(), etof);
  return IPDG_OK;
}

int ipdg_info(ipdg_ctx c, int64_t* out, int n) {
  if (!c || !out) return IPDG_EINVAL;
  // resolved pass-A kernel for lambda = 0 and its launch shape
  const int kern = [&]() -> int { return impl_ops(c->N)->resolve(c, 1, false, nullptr); }();
  const int64_t ksm = kern == 4 ? (int64_t)c->smem_pipe[1][0] : kern == 6 ? (int64_t)c->smem_tpb_m[1] : (int64_t)c->smem[1][0];
  const int64_t kgr = kern == 4 ? c->grid_pipe[1][0] : kern == 6 ? std::min(c->nblocks_t, c->tpb_grid[1][0]) : c->grid[1][0];
  const int64_t v[] = {c->N, c->ref.Np, c->K, c->nblocks, c->E, c->gmax, (int64_t)c->smem[0][0], c->grid[0][0],
                       kern, ksm, kgr};
  for (int i = 0; i < n && i < 11; ++i) out[i] = v[i];
  return IPDG_OK;
}

int64_t ipdg_launch_count(ipdg_ctx c) { return c ? c->launches : -1; }

// debug (not in ipdg.h): per-phase cycle counters of k_sipdg when built with -DIPDG_PHASE_TIMING
int ipdg_debug_phase_cycles(unsigned long long* out8, int reset) {
  if (!out8) return IPDG_EINVAL;
#ifdef IPDG_PHASE_TIMING
  if (cudaMemcpyFromSymbol(out8, ipdg_phase_cycles, 8 * sizeof(unsigned long long)) != cudaSuccess) return IPDG_ECUDA;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(ipdg_phase_cycles, z, sizeof(z)) != cudaSuccess) return IPDG_ECUDA;
  }
#else
  for (int i = 0; i < 8; ++i) out8[i] = 0;
#endif
  return IPDG_OK;
}

// debug (not in ipdg.h): force the split pass A (interior / boundary block lists, odd blocks as
// "boundary") on a single partition, to test the two-launch reduction without a halo.  Re-uploads the
// block lists; call after ipdg_upload_mesh.
int ipdg_debug_split_pass_a(ipdg_ctx c, int on) {
  if (!c || c->K == 0) return IPDG_EINVAL;
  c->force_split = on ? 1 : 0;
  std::vector<int> boff(c->nblocks + 1), goff(c->nblocks + 1);
  CUDA_TRY(c, cudaMemcpy(boff.data(), c->boff, boff.size() * sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(c, cudaMemcpy(goff.data(), c->goff, goff.size() * sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> gid(std::max(1, goff.back()));
  if (goff.back() > 0) CUDA_TRY(c, cudaMemcpy(gid.data(), c->gid, goff.back() * sizeof(int), cudaMemcpyDeviceToHost));
  TRY(build_block_lists(c, c->K, boff, goff, gid));
  TRY(build_tpb(c, c->K, c->etoe_h, c->etof_h, c->pend_bc.data()));
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  c->gkey_x = nullptr;
  return IPDG_OK;
}

// debug (not in ipdg.h): cap every persistent grid at `cap` CTAs (0 = off) so that a small mesh takes
// several element blocks per CTA; applies to the current mesh and every later upload.
int ipdg_debug_grid_cap(ipdg_ctx c, int cap) {
  if (!c || cap < 0) return IPDG_EINVAL;
  c->grid_cap = cap;
  if (c->K > 0) {
    TRY(impl_ops(c->N)->configure(c));
    apply_grid_cap(c);
  }
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  c->gkey_x = nullptr;
  return IPDG_OK;
}

int ipdg_set_variant(ipdg_ctx c, int variant) {
  if (!c || variant < 0 || variant > 6 || variant == 3 || (variant == 5 && c->N > 4)) return IPDG_EINVAL;
  c->variant = variant;
  for (auto& g : c->gexec)
    if (g) { cudaGraphExecDestroy(g); g = nullptr; }
  c->gkey_x = nullptr;
  return IPDG_OK;
}

}  // extern "C"
