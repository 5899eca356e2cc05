// pinn_dd_host.cu -- host orchestration behind the C ABI of include/pinn_dd.h.
//
// Pre-processing stage of Algorithm 1 as it applies to one GPU:
// validate the descriptor, classify every point (residual / training /
// interface), derive 1/N per class and per edge (Eq. 5/6, reading Z2),
// plan tiles and chunks, carve the workspace, and drive the kernels
// K2 (payload) -> K1 (loss + grad) -> K5 (reduce + Adam) on the caller's stream,
// optionally captured once into a CUDA graph.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pinn_dd.h"
#include "pinn_dd_kernels.cuh"
#include "pinn_dd_kernels_tc.cuh"

using namespace pinn;

namespace {

thread_local std::string g_create_error;

// -------------------------------------------------------------------------
// NCCL, resolved at run time (dlopen of libnccl.so.2: the copy the process
// already loaded -- PyTorch's -- is reused, so one NCCL serves both).  Only
// the stable C API below is used (types as in nccl.h).
// -------------------------------------------------------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;            // ncclSuccess = 0
constexpr int kNcclFloat32 = 7;      // ncclFloat32
struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl r;
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) {
      const char* e = dlerror();
      r.why = std::string("dlopen(libnccl.so.2): ") + (e ? e : "not found");
      return r;
    }
    bool all = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(lib, name));
      if (!fn) {
        all = false;
        r.why = std::string("libnccl.so.2 lacks ") + name;
      }
    };
    get(r.GetUniqueId, "ncclGetUniqueId");
    get(r.CommInitRank, "ncclCommInitRank");
    get(r.CommDestroy, "ncclCommDestroy");
    get(r.CommAbort, "ncclCommAbort");
    get(r.Send, "ncclSend");
    get(r.Recv, "ncclRecv");
    get(r.GroupStart, "ncclGroupStart");
    get(r.GroupEnd, "ncclGroupEnd");
    get(r.GetErrorString, "ncclGetErrorString");
    r.ok = all;
    return r;
  }();
  return n;
}

// -------------------------------------------------------------------------
// compiled network shapes
// -------------------------------------------------------------------------
struct Ops {
  int N, NH, DO, ACT;
  int tc;          // 1: hidden layers on the tensor cores (tcgen05 kind::tf32, PINN_DD_FLAG_TF32)
  int pstride;     // Lay::total()
  int P;           // points per tile
  int threads;     // threads per CTA of the fused kernels
  int cps;         // CTAs per SM (persistent grid = cps x #SMs)
  size_t smem;     // dynamic smem of the fused kernel
  void (*k1)(const KArgs&, int grid, size_t smem, cudaStream_t);
  void (*k2)(const KArgs&, int grid, size_t smem, cudaStream_t);
  void (*kf)(const KArgs&, int grid, size_t smem, cudaStream_t);   // fused payload + loss/grad (nullptr: none)
  void (*pred)(const float*, int, float, const float*, const Geo&, int64_t, float*, const int32_t*, cudaStream_t);
  void (*packmap)(std::vector<int32_t>&);
  void (*slopetab)(RArgs&);
  cudaError_t (*setattr)(size_t);
};

template <int N, int NH, int DO, int ACT, int T = kThreads>
struct Inst {
  using C = KCfg<N, NH, DO, T>;
  using LY = Lay<N, NH, DO>;
  static size_t smem() {   // >= 120 KB forces 1 CTA / SM (the CTA owns all of TMEM)
    if constexpr (T == 256)
      return std::max<size_t>(C::SMEM, 120 * 1024);
    else
      return C::SMEM;   // two 128-thread CTAs per SM, 256 TMEM columns each
  }
  static void k1(const KArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_fused<N, NH, DO, ACT, 0, T><<<grid, T, sm, s>>>(a);
  }
  static void k2(const KArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_fused<N, NH, DO, ACT, 1, T><<<grid, T, sm, s>>>(a);
  }
  static void kf(const KArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_fused<N, NH, DO, ACT, 2, T><<<grid, T, sm, s>>>(a);
  }
  static void pred(const float* params, int pstride, float sn, const float* pts, const Geo& geo, int64_t n,
                   float* out, const int32_t* sub_act, cudaStream_t s) {
    const int bs = 128;
    const int64_t g = (n + bs - 1) / bs;
    if (g > 0) k_predict<N, NH, DO, ACT><<<unsigned(g), bs, 0, s>>>(params, pstride, sn, pts, geo, n, out, sub_act);
  }
  // packed index -> internal offset (layer-major W, b, a)
  static void packmap(std::vector<int32_t>& m) {
    m.clear();
    for (int k = 1; k <= NH + 1; ++k) {
      const int nw = LY::nout(k) * LY::nin(k);
      for (int e = 0; e < nw; ++e) m.push_back(LY::offW(k) + e);
      for (int e = 0; e < LY::nout(k); ++e) m.push_back(LY::offB(k) + e);
      if (k <= NH) m.push_back(LY::offA(k));
    }
  }
  static void slopetab(RArgs& r) {
    r.n_hidden = NH;
    for (int k = 1; k <= NH; ++k) {
      r.offW[k - 1] = LY::offW(k);
      r.nW[k - 1] = LY::nout(k) * LY::nin(k);
      r.offB[k - 1] = LY::offB(k);
      r.nB[k - 1] = LY::nout(k);
      r.offA[k - 1] = LY::offA(k);
    }
  }
  static cudaError_t setattr(size_t sm) {
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    const auto carve = cudaFuncAttributePreferredSharedMemoryCarveout;
    cudaError_t e = cudaFuncSetAttribute(k_fused<N, NH, DO, ACT, 0, T>, attr, int(sm));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<N, NH, DO, ACT, 0, T>, carve, 100);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<N, NH, DO, ACT, 1, T>, carve, 100);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<N, NH, DO, ACT, 2, T>, carve, 100);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused<N, NH, DO, ACT, 2, T>, attr, int(sm));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(k_fused<N, NH, DO, ACT, 1, T>, attr, int(sm));
  }
  static Ops ops() {
    static_assert(NH <= kMaxHidden, "too many hidden layers");
    return Ops{N, NH, DO, ACT, 0, LY::total(), C::P, T, C::CPS, smem(), &k1, &k2, &kf, &pred, &packmap, &slopetab,
               &setattr};
  }
};

// tensor-core (TF32) instances of the width-80 shapes: same parameter layout,
// planning and K5 / K6 as the FP32 instance, K1 / K2 / fused step = k_fused_tc
template <int NH, int DO, int ACT>
struct InstTc {
  using F = Inst<80, NH, DO, ACT>;
  using C = tc::TcCfg<NH, DO>;
  static void k1(const KArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_fused_tc<NH, DO, ACT, 0><<<grid, tc::T, sm, s>>>(a);
  }
  static void k2(const KArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_fused_tc<NH, DO, ACT, 1><<<grid, tc::T, sm, s>>>(a);
  }
  static void kf(const KArgs& a, int grid, size_t sm, cudaStream_t s) {
    k_fused_tc<NH, DO, ACT, 2><<<grid, tc::T, sm, s>>>(a);
  }
  static cudaError_t setattr(size_t sm) {
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaFuncSetAttribute(k_fused_tc<NH, DO, ACT, 0>, attr, int(sm));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused_tc<NH, DO, ACT, 1>, attr, int(sm));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_fused_tc<NH, DO, ACT, 2>, attr, int(sm));
    return e;
  }
  static Ops ops() {
    Ops o = F::ops();
    o.tc = 1;
    o.P = tc::P;
    o.threads = tc::T;
    o.cps = 1;
    o.smem = C::SMEM;
    o.k1 = &k1;
    o.k2 = &k2;
    o.kf = &kf;
    o.setattr = &setattr;
    return o;
  }
};

// The shapes of BASELINE.json configs C1-C4 (tanh): 3x20, 5x20, 6x40, 5x80 (D_o = 3);
// C5 (inverse heat, outputs (T, K)): 3x80 with tanh / sin / cos per region (Table 3).
const Ops* find_ops(int N, int NH, int DO, int ACT, int tc) {
  static const Ops table[] = {
      // width 20: two 128-thread CTAs per SM (C3 K1 0.369 -> 0.285 ms)
      Inst<20, 3, 1, 0, 128>::ops(),  Inst<20, 5, 1, 0, 128>::ops(),
      Inst<20, 3, 1, 0>::ops(),       Inst<20, 5, 1, 0>::ops(),
      // width 40: two 128-thread CTAs per SM as well (C2 K1 1.443 -> 1.423 ms since the
      // coalesced chunk-partial read-modify-write; it was 1.65 vs 1.55 ms before)
      Inst<40, 6, 1, 0, 128>::ops(),  Inst<40, 6, 1, 0>::ops(),
      // width 80: one 256-thread CTA per SM (the weights alone are 104 KB of shared memory)
      Inst<80, 5, 3, 0>::ops(),              Inst<80, 3, 2, kActMixed>::ops(),
      // tensor-core hidden layers (PINN_DD_FLAG_TF32)
      InstTc<5, 3, 0>::ops(),                InstTc<3, 2, kActMixed>::ops(),
  };
  // development knob: PINN_DD_CTA_THREADS=128|256 picks the CTA size where both exist
  const char* ev = std::getenv("PINN_DD_CTA_THREADS");
  const int thr = ev ? std::atoi(ev) : 0;
  const Ops* first = nullptr;
  for (const Ops& o : table)
    if (o.N == N && o.NH == NH && o.DO == DO && o.ACT == ACT && o.tc == tc) {
      if (!first) first = &o;
      if (thr == 0 || o.threads == thr) return &o;
    }
  return first;
}

}  // namespace

struct pinn_dd {
  // copied descriptor + owned host arrays
  pinn_dd_desc d;
  std::vector<int32_t> sub_off, n_res, n_data, seg_off, seg_n, norm_counts, act;
  std::vector<int64_t> seg_twin;
  std::vector<float> seg_normal;
  std::vector<pinn_dd_hparams> hp;
  // exchange plan (Algorithm 1 green stage): per peer rank, the local rows sent
  // and the received row range
  std::vector<int32_t> peer_rank;
  std::vector<int64_t> peer_send_off, send_rows, peer_recv_row, peer_recv_n;
  ncclComm_t comm = nullptr;
  cudaStream_t cstream = nullptr;       // exchange stream (forked from / joined to the step's stream)
  cudaEvent_t xfork = nullptr, xjoin = nullptr;
  float* sendbuf = nullptr;
  int32_t* psend = nullptr;
  // peer-store transport (PINN_DD_FLAG_PEER_STORES)
  bool peers_connected = false;
  PeerX px{};
  unsigned long long* xflags = nullptr;   // [kMaxPeers] arrivals here, per peer
  int* xstep = nullptr;                    // fused steps completed
  std::vector<void*> ipc_open;             // peer allocations opened with cudaIpcOpenMemHandle
  // Eq. (4) geometry
  std::vector<float> geo;               // boxes [n_geo][4] or seeds [n_geo][2]
  std::vector<float> poly;              // [n_poly][2]
  std::vector<int32_t> geo_local;       // [n_geo] local subdomain of each geometry entry, -1 = remote
  float* dgeo = nullptr;
  float* dpoly = nullptr;
  int32_t* dgeo_local = nullptr;
  const Ops* ops = nullptr;
  int nf = 0, neq = 0, n_packed = 0, pstride = 0;
  int nsm = 148;
  // plan
  int n_chunks1 = 0, n_chunks2 = 0, grid1 = 0, grid2 = 0, tpc = 1, n_int = 0;
  // device (carved from the workspace)
  float *params = nullptr, *m = nullptr, *v = nullptr, *grad = nullptr;
  float *partial = nullptr, *partial_loss = nullptr, *payload = nullptr, *loss = nullptr;
  float *pinv = nullptr, *gstash = nullptr, *scratch = nullptr;
  int32_t *pinfo = nullptr, *ptwin = nullptr, *sub_chunk = nullptr, *tstep = nullptr, *done = nullptr;
  double* slope_part = nullptr;
  int32_t *sflag = nullptr, *packmap = nullptr, *sub_act = nullptr, *order1 = nullptr, *sched = nullptr;
  int32_t *sub_ctr = nullptr, *sub_tiles = nullptr;
  int sub_list_tiles = 0;      // K1 tiles of all chunks (sticky-schedule heuristic)
  bool sticky_order = false;   // each subdomain's chunks are already in claim order
  float2* segn = nullptr;
  float4 *sub_w = nullptr, *sub_adam = nullptr;
  Chunk *chunks1 = nullptr, *chunks2 = nullptr;
  cudaStream_t stream = nullptr;
  // graph (captured and replayed on an internal stream joined to `stream` by events)
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;
  cudaEvent_t gjoin[2] = {};
  // timing: ev[0..6] step events (see one_iteration), ev[7], ev[8] phased calls;
  // ms = {K2, K1, K5, -, exchange, K1 interior, K1 interface, exposed exchange wait}
  cudaEvent_t ev[9] = {};
  double ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long launches = 0;
  std::string err;
};

namespace {

pinn_dd_status fail(pinn_dd* h, pinn_dd_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h)
    h->err = buf;
  else
    g_create_error = buf;
  return s;
}

#define CK(h, call)                                                                                         \
  do {                                                                                                      \
    cudaError_t e_ = (call);                                                                                \
    if (e_ != cudaSuccess) return fail(h, PINN_DD_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                                  \
  } while (0)

int n_eq_of(int pde) { return pde == PINN_DD_PDE_NS ? 3 : 1; }

// Tiles per full chunk of a run of `cnt` points: at most ~148 chunks per run
// (one per SM, so that ONE subdomain alone -- a GPU's share under strong
// scaling at 8 GPUs -- still fills the persistent grid: C4 at 8 GPUs 126 ->
// 148 chunks; 296 measured 4 % slower at 1 GPU; 1024 for giant runs, below).
// Runs of >= 200 tiles use chunks of >= m tiles, m = ACC / 2048 clamped to
// [1, 4] (ACC = floats of a chunk's gradient partial, flushed once per chunk
// and read back by K5a: 6x40 -> 4, 5x20 -> 1, i.e. 3-tile chunks for C3's
// 324-tile runs, K1 0.267 -> 0.260 ms); shorter runs (the small C5 regions)
// 2-tile chunks (with the sticky queues of the fused step, which keep a CTA on
// one region, 2-tile chunks halve the per-chunk work: C5 K1 0.438 -> 0.430
// ms, TF32 0.221 -> 0.218 ms, and keeping 1-tile interface chunks cost TF32
// 7 %; on the global queue 1-tile chunks had the shorter tail: 0.573 -> 0.531
// ms in round 1).  Depends only on cnt and the net (placement invariance).
int chunk_tiles(int cnt, int P, int acc, bool interior = true) {
  static const int min_env = [] {   // development knob: PINN_DD_MIN_CHUNK_TILES
    const char* e = std::getenv("PINN_DD_MIN_CHUNK_TILES");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int tiles = (cnt + P - 1) / P;
  const int m = std::min(4, std::max(1, acc / 2048));
  // a small-partial net (m = 1: width 20) with runs of at most two waves of
  // the 296 CTA slots of its 128-thread instance takes one-tile chunks
  // (interface runs included): the C3 weak-scaling subdomain (20k points, 315
  // tiles) then spreads over every slot instead of 105 three-tile chunks
  // (step 77.0 -> 69.5 us; C3 x 8 per GPU 0.272 -> 0.274 ms, its K5 reads 3x
  // the partials; with 2-tile interface chunks it was 0.293 ms)
  if (!min_env && m == 1 && tiles <= 2 * 296) return 1;
  const int min_tiles = min_env ? min_env : (tiles >= 200 ? m : 2);
  (void)interior;
  // a giant run (the data-parallel comparator's single subdomain: 7,530 tiles
  // of 32) would get only ~128 chunks -- fewer than the persistent CTAs -- so
  // runs of > 2048 tiles with partials of <= 64 KB may use up to 1024 chunks
  static const int maxc_env = [] {   // development knob: PINN_DD_MAX_CHUNKS
    const char* e = std::getenv("PINN_DD_MAX_CHUNKS");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int max_chunks = maxc_env ? maxc_env : ((tiles > 2048 && acc <= 16384) ? 1024 : 148);
  return std::max(min_tiles, (tiles + max_chunks - 1) / max_chunks);
}

// point counts of the K1 chunks of a run of `cnt` points: full chunks of
// chunk_tiles(cnt) tiles, the remainder as one-tile chunks (the schedule's
// tail); depends only on cnt (placement invariance)
void chunk_sizes(int cnt, int P, int acc, bool interior, std::vector<int>& out) {
  if (cnt == 0) return;
  const int span = chunk_tiles(cnt, P, acc, interior) * P;
  int s0 = 0;
  for (; s0 + span <= cnt; s0 += span) out.push_back(span);
  for (; s0 < cnt; s0 += P) out.push_back(std::min(P, cnt - s0));
}

// K1 chunks of a subdomain: its `na` residual + training points, then its `ni`
// interface points (a chunk never mixes the two, so the interface part can run
// after the payload exchange); sign of the entry = interface run.
// An empty subdomain still gets one (empty) chunk and thus a partial slot.
std::vector<int> split_chunks(int na, int ni, int P, int acc) {
  std::vector<int> a, b;
  chunk_sizes(na, P, acc, true, a);
  chunk_sizes(ni, P, acc, false, b);
  for (int& v : b) v = -v - 1;
  a.insert(a.end(), b.begin(), b.end());
  if (a.empty()) a.push_back(0);
  return a;
}

struct Carve {
  size_t off = 0;
  template <class T>
  size_t take(size_t count) {
    size_t o = off;
    off += (count * sizeof(T) + 255) & ~size_t(255);
    return o;
  }
};

struct Layout {
  size_t params, m, v, grad, scratch, partial, ploss, payload, pinfo, pinv, ptwin, segn, subw, suba, subact, ch1, ord1,
      sched, ch2, subch, sctr, stiles,
      tstep, done, sflag, loss, packmap, slopep, sendbuf, psend, dgeo, dpoly, dgeoloc, xflags, xstep, gstash,
      total;
};

// validation + planning shared by workspace_size and create
pinn_dd_status plan(const pinn_dd_desc* d, pinn_dd* h, Layout* L, int nsm) {
  if (!d) return fail(h, PINN_DD_EINVAL, "desc is NULL");
  if (d->d_in != 2) return fail(h, PINN_DD_EINVAL, "d_in must be 2 (got %d)", d->d_in);
  if (d->method < 0 || d->method > 3) return fail(h, PINN_DD_EINVAL, "bad method %d", d->method);
  if (d->pde < 0 || d->pde > 4) return fail(h, PINN_DD_EINVAL, "bad pde %d", d->pde);
  const int want_do = d->pde == PINN_DD_PDE_NS ? 3 : (d->pde == PINN_DD_PDE_HEAT_INV ? 2 : 1);
  if (d->d_out != want_do) return fail(h, PINN_DD_EINVAL, "d_out %d does not match pde %d", d->d_out, d->pde);
  if (d->activation < 0 || d->activation > 2) return fail(h, PINN_DD_EINVAL, "bad activation %d", d->activation);
  bool mixed = false;
  if (d->sub_activation) {
    if (d->n_sub < 1) return fail(h, PINN_DD_EINVAL, "n_sub must be >= 1");
    for (int q = 0; q < d->n_sub; ++q) {
      if (d->sub_activation[q] < 0 || d->sub_activation[q] > 2)
        return fail(h, PINN_DD_EINVAL, "subdomain %d: bad activation %d", q, d->sub_activation[q]);
      mixed |= d->sub_activation[q] != d->sub_activation[0];
    }
  }
  const int act0 = d->sub_activation ? d->sub_activation[0] : d->activation;
  // one compiled activation if uniform, else the per-subdomain (kActMixed) instance
  const int tc = (d->flags & PINN_DD_FLAG_TF32) ? 1 : 0;
  if (tc && (d->flags & PINN_DD_FLAG_GLOBAL_STASH))
    return fail(h, PINN_DD_EUNSUPPORTED, "PINN_DD_FLAG_TF32 keeps its stash in TMEM (no global stash)");
  const Ops* ops = mixed ? nullptr : find_ops(d->width, d->n_hidden, d->d_out, act0, tc);
  if (!ops) ops = find_ops(d->width, d->n_hidden, d->d_out, kActMixed, tc);
  if (!ops)
    return fail(h, PINN_DD_EUNSUPPORTED, "network [2, %dx%d, %d] activation %d%s%s not compiled in", d->width,
                d->n_hidden, d->d_out, act0, mixed ? " (mixed per subdomain)" : "",
                tc ? " with tensor-core (TF32) layers" : "");
  if (d->n_sub < 1) return fail(h, PINN_DD_EINVAL, "n_sub must be >= 1");
  if (!d->sub_point_offset || !d->sub_n_res || !d->sub_n_data || !d->sub_seg_offset || !d->sub_hparams)
    return fail(h, PINN_DD_EINVAL, "subdomain arrays must not be NULL");
  if (d->n_seg > 0 && (!d->seg_n || !d->seg_normal || !d->seg_twin))
    return fail(h, PINN_DD_EINVAL, "segment arrays must not be NULL");
  if (d->method == PINN_DD_METHOD_PINN && d->n_seg != 0)
    return fail(h, PINN_DD_EINVAL, "method PINN has no interfaces");
  if (d->n_points < 0 || d->n_recv < 0) return fail(h, PINN_DD_EINVAL, "negative counts");
  if (d->n_points > 0 && !d->coords) return fail(h, PINN_DD_EINVAL, "coords is NULL");
  if (d->n_points >= (int64_t(1) << 31) || d->n_points + d->n_recv >= (int64_t(1) << 31))
    return fail(h, PINN_DD_EINVAL, "too many points for int32 indexing");
  if (d->sub_point_offset[0] != 0 || d->sub_seg_offset[0] != 0)
    return fail(h, PINN_DD_EINVAL, "offsets must start at 0");
  if (d->sub_point_offset[d->n_sub] != d->n_points)
    return fail(h, PINN_DD_EINVAL, "sub_point_offset[n_sub] != n_points");
  if (d->sub_seg_offset[d->n_sub] != d->n_seg) return fail(h, PINN_DD_EINVAL, "sub_seg_offset[n_sub] != n_seg");
  if (d->sub_norm_counts)
    for (int q = 0; q < d->n_sub; ++q)
      if (d->sub_norm_counts[2 * q] < d->sub_n_res[q] || d->sub_norm_counts[2 * q + 1] < d->sub_n_data[q] ||
          (d->sub_n_res[q] > 0 && d->sub_norm_counts[2 * q] <= 0) ||
          (d->sub_n_data[q] > 0 && d->sub_norm_counts[2 * q + 1] <= 0))
        return fail(h, PINN_DD_EINVAL, "subdomain %d: normalisation counts below the local counts", q);
  bool any_data = false;
  for (int q = 0; q < d->n_sub; ++q) {
    const int64_t cnt = int64_t(d->sub_point_offset[q + 1]) - d->sub_point_offset[q];
    if (cnt < 0 || d->sub_n_res[q] < 0 || d->sub_n_data[q] < 0)
      return fail(h, PINN_DD_EINVAL, "subdomain %d: negative count", q);
    if (d->sub_seg_offset[q + 1] < d->sub_seg_offset[q])
      return fail(h, PINN_DD_EINVAL, "subdomain %d: seg offsets not monotone", q);
    int64_t ni = 0;
    for (int s = d->sub_seg_offset[q]; s < d->sub_seg_offset[q + 1]; ++s) {
      if (d->seg_n[s] < 1) return fail(h, PINN_DD_EINVAL, "segment %d: N_I must be >= 1", s);
      ni += d->seg_n[s];
    }
    if (d->sub_n_res[q] + d->sub_n_data[q] + ni != cnt)
      return fail(h, PINN_DD_EINVAL, "subdomain %d: N_F + N_u + sum N_I = %lld != %lld points", q,
                  (long long)(d->sub_n_res[q] + d->sub_n_data[q] + ni), (long long)cnt);
    if (d->sub_n_data[q] > 0) any_data = true;
  }
  if (any_data && (!d->target || !d->mask)) return fail(h, PINN_DD_EINVAL, "target/mask NULL with training points");
  for (int s = 0; s < d->n_seg; ++s) {
    const float n1 = d->seg_normal[2 * s], n2 = d->seg_normal[2 * s + 1];
    if (std::fabs(n1 * n1 + n2 * n2 - 1.0f) > 1e-5f) return fail(h, PINN_DD_EINVAL, "segment %d: normal not unit", s);
    if (d->method == PINN_DD_METHOD_CPINN && d->pde == PINN_DD_PDE_BURGERS && n2 != 0.0f)
      return fail(h, PINN_DD_EINVAL,
                  "cPINN with a time-axis interface (segment %d) is not allowed (P:816, SPEC.md:689)", s);
    const int64_t tw = d->seg_twin[s];
    if (tw < 0 || tw + d->seg_n[s] > d->n_points + d->n_recv)
      return fail(h, PINN_DD_EPROTOCOL, "segment %d: twin rows [%lld, +%d) out of range", s, (long long)tw,
                  d->seg_n[s]);
  }
  // exchange plan: peers' received ranges tile [n_points, n_points + n_recv)
  // in peer order; sent rows are local interface points (checked in create)
  if (d->n_peers < 0 || (d->n_peers > 0 && (!d->peer_rank || !d->peer_send_off || !d->peer_recv_row ||
                                            !d->peer_recv_n || (!d->send_rows && d->peer_send_off[d->n_peers] > 0))))
    return fail(h, PINN_DD_EPROTOCOL, "exchange plan arrays must not be NULL (n_peers = %d)", d->n_peers);
  int64_t n_send = 0;
  {
    int64_t row = d->n_points;
    if (d->n_peers > 0 && d->peer_send_off[0] != 0) return fail(h, PINN_DD_EPROTOCOL, "peer_send_off[0] != 0");
    for (int i = 0; i < d->n_peers; ++i) {
      if (i > 0 && d->peer_rank[i] <= d->peer_rank[i - 1])
        return fail(h, PINN_DD_EPROTOCOL, "peer ranks must be distinct and ascending");
      if (d->nccl_id && (d->peer_rank[i] < 0 || d->peer_rank[i] >= d->world))
        return fail(h, PINN_DD_EPROTOCOL, "peer rank %d outside the communicator of %d", d->peer_rank[i], d->world);
      if (d->peer_send_off[i + 1] < d->peer_send_off[i])
        return fail(h, PINN_DD_EPROTOCOL, "peer_send_off not monotone");
      if (d->peer_recv_row[i] != row || d->peer_recv_n[i] < 0)
        return fail(h, PINN_DD_EPROTOCOL, "peer %d: received rows must start at %lld", i, (long long)row);
      row += d->peer_recv_n[i];
    }
    if (row != d->n_points + d->n_recv)
      return fail(h, PINN_DD_EPROTOCOL, "received rows cover %lld of n_recv = %lld", (long long)(row - d->n_points),
                  (long long)d->n_recv);
    if (d->n_peers > 0) n_send = d->peer_send_off[d->n_peers];
    for (int64_t j = 0; j < n_send; ++j)
      if (d->send_rows[j] < 0 || d->send_rows[j] >= d->n_points)
        return fail(h, PINN_DD_EPROTOCOL, "send row %lld out of range", (long long)d->send_rows[j]);
  }
  if (d->nccl_id && (d->world < 1 || d->rank < 0 || d->rank >= d->world))
    return fail(h, PINN_DD_EINVAL, "rank %d / world %d", d->rank, d->world);
  if (d->flags & PINN_DD_FLAG_PEER_STORES) {
    if (d->nccl_id) return fail(h, PINN_DD_EINVAL, "PINN_DD_FLAG_PEER_STORES and nccl_id are exclusive");
    if (d->n_peers > kMaxPeers) return fail(h, PINN_DD_EUNSUPPORTED, "peer stores: at most %d peers", kMaxPeers);
  }
  // Eq. (4) geometry
  if (d->geometry < 0 || d->geometry > 2) return fail(h, PINN_DD_EINVAL, "bad geometry %d", d->geometry);
  if (d->geometry != PINN_DD_GEOM_NONE) {
    if (d->n_geo < 1 || !d->geo || !d->geo_local) return fail(h, PINN_DD_EINVAL, "geometry arrays must not be NULL");
    if (d->geometry == PINN_DD_GEOM_VORONOI && (d->n_poly < 3 || !d->poly))
      return fail(h, PINN_DD_EINVAL, "Voronoi geometry needs a polygon of >= 3 vertices");
    if (!(d->geo_tol >= 0.0f)) return fail(h, PINN_DD_EINVAL, "geo_tol must be >= 0");
    for (int g = 0; g < d->n_geo; ++g)
      if (d->geo_local[g] < -1 || d->geo_local[g] >= d->n_sub)
        return fail(h, PINN_DD_EINVAL, "geo_local[%d] = %d out of range", g, d->geo_local[g]);
  }
  // tiles and chunks.  The chunking of a subdomain depends only on its own
  // point count (never on which other subdomains share the GPU), so the
  // fixed-order reduction is bitwise placement-invariant.
  const int P = ops->P;
  int n1 = 0, n2 = 0;
  std::vector<int> sizes;
  for (int q = 0; q < d->n_sub; ++q) {
    const int cnt = d->sub_point_offset[q + 1] - d->sub_point_offset[q];
    const int na = d->sub_n_res[q] + d->sub_n_data[q];
    n1 += int(split_chunks(na, cnt - na, P, ops->pstride).size());
    const int ni = cnt - d->sub_n_res[q] - d->sub_n_data[q];
    n2 += (ni + P - 1) / P;
  }
  const int pstride = ops->pstride;
  const int nf = d->d_out + n_eq_of(d->pde);
  const size_t ns = size_t(d->n_sub);
  const size_t npt = size_t(d->n_points);
  const int grid1 = std::min(n1, nsm * ops->cps);
  Carve c;
  L->params = c.take<float>(ns * pstride);
  L->m = c.take<float>(ns * pstride);
  L->v = c.take<float>(ns * pstride);
  L->grad = c.take<float>(ns * pstride);
  L->scratch = c.take<float>(ns * pstride);
  L->partial = c.take<float>(size_t(n1) * pstride);
  L->ploss = c.take<float>(size_t(n1) * 4);
  // peer stores alternate two receive slots by step parity
  const size_t nslots = (d->flags & PINN_DD_FLAG_PEER_STORES) ? 2 : 1;
  L->payload = c.take<float>((npt + nslots * size_t(d->n_recv) + 1) * nf);
  L->pinfo = c.take<int32_t>(npt + 1);
  L->pinv = c.take<float>(npt + 1);
  L->ptwin = c.take<int32_t>(npt + 1);
  L->segn = c.take<float2>(size_t(d->n_seg) + 1);
  L->subw = c.take<float4>(ns);
  L->subact = c.take<int32_t>(ns);
  L->suba = c.take<float4>(ns);
  L->ch1 = c.take<Chunk>(size_t(n1));
  L->ord1 = c.take<int32_t>(size_t(2 * n1));   // [all | interior, interface] processing orders
  L->sched = c.take<int32_t>(8);   // [0,1] K1, [2,3] K2, [4] fused step: payload chunks done
  L->ch2 = c.take<Chunk>(size_t(n2) + 1);
  L->subch = c.take<int32_t>(ns + 1);
  L->tstep = c.take<int32_t>(ns);
  L->done = c.take<int32_t>(ns);
  L->sflag = c.take<int32_t>(ns);
  L->loss = c.take<float>(ns * 8);
  L->packmap = c.take<int32_t>(size_t(pstride));
  L->slopep = c.take<double>(ns * size_t((pstride + kRW - 1) / kRW) * kMaxHidden);
  L->sendbuf = c.take<float>(size_t(n_send + 1) * nf);
  L->psend = c.take<int32_t>(npt + 1);
  const int ngeo = d->geometry ? d->n_geo : 0;
  L->dgeo = c.take<float>(size_t(ngeo) * 4 + 4);
  L->dpoly = c.take<float>(size_t(d->geometry == PINN_DD_GEOM_VORONOI ? d->n_poly : 0) * 2 + 2);
  L->dgeoloc = c.take<int32_t>(size_t(ngeo) + 1);
  L->xflags = c.take<unsigned long long>(kMaxPeers);
  L->xstep = c.take<int32_t>(1);
  // fused step's per-subdomain chunk queues (sticky schedule)
  L->sctr = c.take<int32_t>(ns);
  L->stiles = c.take<int32_t>(ns + 1);
  L->gstash = (d->flags & PINN_DD_FLAG_GLOBAL_STASH)
                  ? c.take<float>(size_t(grid1) * d->n_hidden * kA * ops->threads)
                  : c.off;
  L->total = c.off;
  if (h) {
    h->ops = ops;
    h->tpc = chunk_tiles(d->n_sub ? d->sub_point_offset[1] - d->sub_point_offset[0] : 0, P, ops->pstride);
    h->n_chunks1 = n1;
    h->n_chunks2 = n2;
    h->grid1 = grid1;
    h->grid2 = std::max(1, std::min(n2, nsm * ops->cps));
    h->pstride = pstride;
    h->nf = nf;
    h->neq = n_eq_of(d->pde);
  }
  return PINN_DD_OK;
}

int device_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

KArgs make_kargs(pinn_dd* h, bool payload_tiles) {
  KArgs a;
  const pinn_dd_desc& d = h->d;
  a.coords = d.coords;
  a.target = d.target;
  a.mask = d.mask;
  a.pinfo = h->pinfo;
  a.pinv = h->pinv;
  a.ptwin = h->ptwin;
  a.seg_normal = h->segn;
  a.params = h->params;
  a.sub_w = h->sub_w;
  a.sub_act = h->sub_act;
  a.chunks = payload_tiles ? h->chunks2 : h->chunks1;
  a.chunks2 = nullptr;
  a.n_chunks2 = 0;
  a.order = payload_tiles ? nullptr : h->order1;   // launch_k1 selects the part
  a.sub_chunk_off = nullptr;                       // launch_fused: sticky queues
  a.sub_ctr = nullptr;
  a.sub_tiles = nullptr;
  a.n_sub = d.n_sub;
  a.sched = h->sched + (payload_tiles ? 2 : 0);
  a.n_chunks = payload_tiles ? h->n_chunks2 : h->n_chunks1;
  a.n_points = d.n_points;
  a.pstride = h->pstride;
  a.partial = h->partial;
  a.partial_loss = h->partial_loss;
  a.payload = h->payload;
  a.psend = h->send_rows.empty() ? nullptr : h->psend;
  a.sendbuf = h->sendbuf;
  a.px = h->px;
  a.px.n = 0;   // only the fused step stores into peers (launch_fused)
  a.gstash = (d.flags & PINN_DD_FLAG_GLOBAL_STASH) ? h->gstash : nullptr;
  a.pc.pde = d.pde;
  a.pc.nu = d.nu;
  a.pc.re = d.re;
  a.method = d.method;
  a.slope_n = d.slope_n;
  // S of Delta_S: Burgers needs u_xx only (x1); the 2-D operators need both
  a.m1 = 1.0f;
  a.m2 = d.pde == PINN_DD_PDE_BURGERS ? 0.0f : 1.0f;
  return a;
}

RArgs make_rargs(pinn_dd* h, int mode) {
  RArgs r;
  r.partial = h->partial;
  r.partial_loss = h->partial_loss;
  r.sub_chunk = h->sub_chunk;
  r.pstride = h->pstride;
  r.grad = h->grad;
  r.params = h->params;
  r.m = h->m;
  r.v = h->v;
  r.tstep = h->tstep;
  r.done = h->done;
  r.sub_w = h->sub_w;
  r.sub_adam = h->sub_adam;
  r.loss = h->loss;
  r.sflag = h->sflag;
  r.slope_part = h->slope_part;
  r.mode = mode;
  r.nb5a = (h->pstride + kRW - 1) / kRW;
  h->ops->slopetab(r);
  return r;
}

pinn_dd_status launch_k2(pinn_dd* h) {
  if (h->n_chunks2 == 0) return PINN_DD_OK;
  h->ops->k2(make_kargs(h, true), h->grid2, h->ops->smem, h->stream);
  ++h->launches;
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}
// part 0: every K1 chunk; 1: residual + training chunks; 2: interface chunks
pinn_dd_status launch_k1(pinn_dd* h, int part = 0) {
  KArgs a = make_kargs(h, false);
  const int n1 = h->n_chunks1;
  if (part == 1) {
    a.order = h->order1 + n1;
    a.n_chunks = h->n_int;
  } else if (part == 2) {
    a.order = h->order1 + n1 + h->n_int;
    a.n_chunks = n1 - h->n_int;
  }
  if (a.n_chunks == 0) return PINN_DD_OK;
  h->ops->k1(a, std::min(h->grid1, a.n_chunks), h->ops->smem, h->stream);
  ++h->launches;
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}
// mode 0: reduce + slopes (loss_grad); 1: reduce + slopes + Adam (step);
// 2: Adam on the stored gradient (pinn_dd_adam)
// K5a with 512-thread blocks for nets of at most this many partial floats
// (width 20: C3's weak-scaling subdomain, 315 one-tile chunk partials over 14
// entry blocks)
constexpr int kSmallNet = 4096;
pinn_dd_status launch_k5(pinn_dd* h, int mode) {
  dim3 g((h->pstride + kRB - 1) / kRB, h->d.n_sub);
  if (mode != 2) {
    // status bits of this evaluation start at 0 (zeroed at create and by the K5b that published the last ones)
    const dim3 g5a((h->pstride + kRW - 1) / kRW, h->d.n_sub);
    if (h->pstride <= kSmallNet)
      k_reduce<512><<<g5a, 512, 0, h->stream>>>(make_rargs(h, 0));
    else
      k_reduce<kRB><<<g5a, kRB, 0, h->stream>>>(make_rargs(h, 0));
    ++h->launches;
    CK(h, cudaGetLastError());
  }
  RArgs r = make_rargs(h, mode);   // 2: Adam on the stored gradient (slopes were filled by loss_grad)
  k_slope_adam<<<g, kRB, 0, h->stream>>>(r);
  ++h->launches;
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}

// record = event timestamps around K2 / K1 / K5 (as external event-record
// nodes when captured into the step graph)
pinn_dd_status record(pinn_dd* h, int i, bool capturing, cudaStream_t st = nullptr) {
  if (!st) st = h->stream;
  if (capturing)
    CK(h, cudaEventRecordWithFlags(h->ev[i], st, cudaEventRecordExternal));
  else
    CK(h, cudaEventRecord(h->ev[i], st));
  return PINN_DD_OK;
}

float elapsed(pinn_dd* h, int a, int b) {
  float ms = 0.0f;
  return cudaEventElapsedTime(&ms, h->ev[a], h->ev[b]) == cudaSuccess ? ms : 0.0f;
}

// kind 0: K2 -> K1 -> K5 (events 0..3); 1: fused K2+K1 -> K5 (1..3);
// 2: distributed (0..6, see one_iteration)
pinn_dd_status accumulate_times(pinn_dd* h, int kind) {
  CK(h, cudaEventSynchronize(h->ev[3]));
  if (kind == 2) {
    h->ms[0] += elapsed(h, 0, 1);
    const double in = elapsed(h, 1, 2), ifc = elapsed(h, 6, 5);
    h->ms[1] += in + ifc;
    h->ms[2] += elapsed(h, 5, 3);
    h->ms[4] += elapsed(h, 1, 4);
    h->ms[5] += in;
    h->ms[6] += ifc;
    h->ms[7] += elapsed(h, 2, 6);
    return PINN_DD_OK;
  }
  if (kind == 0) h->ms[0] += elapsed(h, 0, 1);
  h->ms[1] += elapsed(h, 1, 2);
  h->ms[2] += elapsed(h, 2, 3);
  return PINN_DD_OK;
}

// K2 and K1 as one persistent launch (payload chunks first, interface loss
// chunks wait on the payload-done counter); all twins must be local
pinn_dd_status launch_fused(pinn_dd* h) {
  KArgs a = make_kargs(h, false);
  a.chunks2 = h->chunks2;
  a.n_chunks2 = h->n_chunks2;
  // loss chunks: residual + training chunks (big first), then the interface
  // chunks, so that no CTA waits on the payload counter while interior work
  // is left (C5's one-tile chunks interleaved them: 5 % of K1's samples were
  // the payload wait)
  a.order = h->order1 + h->n_chunks1;
  // sticky per-subdomain queues (development A/B knob PINN_DD_NO_STICKY=1)
  // Only where a CTA runs many small chunks (C5's one-tile chunks: K1 0.470
  // -> 0.462 ms, TF32 0.358 -> 0.272 ms): with 4-tile chunks (C2: 8 per CTA)
  // the per-subdomain queues lose the global largest-first tail balance (C2
  // K1 1.345 -> 1.450 ms).
  static const bool no_sticky = std::getenv("PINN_DD_NO_STICKY") != nullptr;
  if (!no_sticky && h->sticky_order && h->n_chunks1 >= 4 * h->grid1 && h->sub_list_tiles <= 2 * h->n_chunks1) {
    a.sub_chunk_off = h->sub_chunk;
    a.sub_ctr = h->sub_ctr;
    a.sub_tiles = h->sub_tiles;
  }
  if (h->peers_connected) a.px = h->px;
  h->ops->kf(a, std::min(h->grid1, a.n_chunks + a.n_chunks2), h->ops->smem, h->stream);
  ++h->launches;
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}

// remote twins exchanged by NCCL (or the caller); peer stores run in the fused launch
bool remote(const pinn_dd* h) { return !h->peer_rank.empty() && !h->peers_connected; }

bool use_fused(const pinn_dd* h) {
  static const bool off = std::getenv("PINN_DD_NO_FUSED_STEP") != nullptr;   // development A/B knob
  if (h->peers_connected) return true;
  return h->ops->kf && h->n_chunks2 > 0 && h->d.n_recv == 0 && !remote(h) && !off;
}

#define CKN(h, call)                                                                                         \
  do {                                                                                                       \
    const ncclResult_t r_ = (call);                                                                          \
    if (r_ != 0) return fail(h, PINN_DD_ENCCL, "%s: %s", #call, nccl().GetErrorString(r_));                 \
  } while (0)

// the green stage on stream `st`: one NCCL group of every peer's send (the
// rows K2 wrote to the send buffer) and receive (straight into the payload
// buffer's received rows)
pinn_dd_status nccl_group(pinn_dd* h, cudaStream_t st) {
  const Nccl& N = nccl();
  const size_t nf = size_t(h->nf);
  CKN(h, N.GroupStart());
  for (size_t i = 0; i < h->peer_rank.size(); ++i) {
    const int64_t s0 = h->peer_send_off[i], sn = h->peer_send_off[i + 1] - s0;
    if (sn > 0) CKN(h, N.Send(h->sendbuf + size_t(s0) * nf, size_t(sn) * nf, kNcclFloat32, h->peer_rank[i], h->comm, st));
    if (h->peer_recv_n[i] > 0)
      CKN(h, N.Recv(h->payload + size_t(h->peer_recv_row[i]) * nf, size_t(h->peer_recv_n[i]) * nf, kNcclFloat32,
                    h->peer_rank[i], h->comm, st));
  }
  CKN(h, N.GroupEnd());
  return PINN_DD_OK;
}

pinn_dd_status one_iteration(pinn_dd* h, bool timed, bool capturing) {
  pinn_dd_status s;
  if (remote(h)) {
    // Algorithm 1 with remote neighbours: K2 -> [exchange stream: NCCL group]
    // || K1 over residual + training points -> wait -> K1 over interface
    // points -> K5.  Events: 0 before K2, 1 after K2, 4 exchange done (exchange
    // stream), 2 after K1 interior, 6 after the wait, 5 after K1 interface, 3 after K5.
    if (timed && (s = record(h, 0, capturing)) != PINN_DD_OK) return s;
    if ((s = launch_k2(h)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 1, capturing)) != PINN_DD_OK) return s;
    CK(h, cudaEventRecord(h->xfork, h->stream));
    CK(h, cudaStreamWaitEvent(h->cstream, h->xfork, 0));
    if ((s = nccl_group(h, h->cstream)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 4, capturing, h->cstream)) != PINN_DD_OK) return s;
    CK(h, cudaEventRecord(h->xjoin, h->cstream));
    if ((s = launch_k1(h, 1)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 2, capturing)) != PINN_DD_OK) return s;
    CK(h, cudaStreamWaitEvent(h->stream, h->xjoin, 0));
    if (timed && (s = record(h, 6, capturing)) != PINN_DD_OK) return s;
    if ((s = launch_k1(h, 2)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 5, capturing)) != PINN_DD_OK) return s;
    if ((s = launch_k5(h, 1)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 3, capturing)) != PINN_DD_OK) return s;
    if (timed && !capturing) return accumulate_times(h, 2);
    return PINN_DD_OK;
  }
  if (timed && !use_fused(h) && (s = record(h, 0, capturing)) != PINN_DD_OK) return s;
  if (use_fused(h)) {
    // K2 folded into K1 (reported as 0 ms); three event nodes, not four: each
    // event-record node costs ~2.7 us of step latency on the B200
    if (timed && (s = record(h, 1, capturing)) != PINN_DD_OK) return s;
    if ((s = launch_fused(h)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 2, capturing)) != PINN_DD_OK) return s;
    if ((s = launch_k5(h, 1)) != PINN_DD_OK) return s;
    if (timed && (s = record(h, 3, capturing)) != PINN_DD_OK) return s;
    if (timed && !capturing) return accumulate_times(h, 1);
    return PINN_DD_OK;
  }
  if ((s = launch_k2(h)) != PINN_DD_OK) return s;
  if (timed && (s = record(h, 1, capturing)) != PINN_DD_OK) return s;
  if ((s = launch_k1(h)) != PINN_DD_OK) return s;
  if (timed && (s = record(h, 2, capturing)) != PINN_DD_OK) return s;
  if ((s = launch_k5(h, 1)) != PINN_DD_OK) return s;
  if (timed && (s = record(h, 3, capturing)) != PINN_DD_OK) return s;
  if (timed && !capturing) return accumulate_times(h, 0);
  return PINN_DD_OK;
}

int timing_kind(const pinn_dd* h) { return remote(h) ? 2 : (use_fused(h) ? 1 : 0); }

// launches per iteration (as counted by the graph replay)
int iteration_launches(const pinn_dd* h) {
  if (remote(h)) return (h->n_chunks2 > 0) + (h->n_int > 0) + (h->n_chunks1 - h->n_int > 0) + 2;
  return use_fused(h) ? 3 : (h->n_chunks2 > 0 ? 4 : 3);
}

// loss column 5 holds the status bits of the last evaluation (kFlag*)
pinn_dd_status check_status(pinn_dd* h, const float* loss_host) {
  for (int q = 0; q < h->d.n_sub; ++q) {
    const int f = int(loss_host[q * 8 + 5]);
    if (f & kFlagJ) return fail(h, PINN_DD_ENONFINITE, "non-finite J in subdomain %d", q);
    if (f & kFlagGrad) return fail(h, PINN_DD_ENONFINITE, "non-finite W/b gradient in subdomain %d", q);
    if (f & kFlagSlopeZero)
      return fail(h, PINN_DD_ENONFINITE, "slope a^k = 0 in subdomain %d: its gradient is undefined (NaN)", q);
    if (f & kFlagSlopeGrad) return fail(h, PINN_DD_ENONFINITE, "non-finite slope gradient in subdomain %d", q);
  }
  return PINN_DD_OK;
}

}  // namespace

extern "C" {

int64_t pinn_dd_n_params(int32_t d_in, int32_t width, int32_t n_hidden, int32_t d_out) {
  if (d_in < 1 || width < 1 || n_hidden < 1 || d_out < 1) return -1;
  int64_t n = int64_t(width) * d_in + width + 1;
  n += int64_t(n_hidden - 1) * (int64_t(width) * width + width + 1);
  n += int64_t(d_out) * width + d_out;
  return n;
}

pinn_dd_status pinn_dd_workspace_size(const pinn_dd_desc* d, size_t* bytes) {
  if (!bytes) return fail(nullptr, PINN_DD_EINVAL, "bytes is NULL");
  Layout L;
  pinn_dd_status s = plan(d, nullptr, &L, device_sms());
  if (s != PINN_DD_OK) return s;
  *bytes = L.total;
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_create(const pinn_dd_desc* d, void* ws, size_t ws_bytes, pinn_dd** out) {
  if (!out) return fail(nullptr, PINN_DD_EINVAL, "out is NULL");
  *out = nullptr;
  pinn_dd* h = new pinn_dd();
  Layout L;
  h->nsm = device_sms();
  pinn_dd_status s = plan(d, h, &L, h->nsm);
  if (s != PINN_DD_OK) {
    g_create_error = h->err;
    delete h;
    return s;
  }
  if (!ws || ws_bytes < L.total || (reinterpret_cast<uintptr_t>(ws) & 255u)) {
    fail(nullptr, PINN_DD_EINVAL, "workspace %p of %zu bytes; need %zu bytes, 256-B aligned", ws, ws_bytes, L.total);
    delete h;
    return PINN_DD_EINVAL;
  }
  // deep copies of the host arrays
  h->d = *d;
  const int ns = d->n_sub;
  h->sub_off.assign(d->sub_point_offset, d->sub_point_offset + ns + 1);
  h->n_res.assign(d->sub_n_res, d->sub_n_res + ns);
  h->n_data.assign(d->sub_n_data, d->sub_n_data + ns);
  h->seg_off.assign(d->sub_seg_offset, d->sub_seg_offset + ns + 1);
  h->hp.assign(d->sub_hparams, d->sub_hparams + ns);
  if (d->sub_norm_counts) h->norm_counts.assign(d->sub_norm_counts, d->sub_norm_counts + 2 * ns);
  if (d->n_seg > 0) {
    h->seg_n.assign(d->seg_n, d->seg_n + d->n_seg);
    h->seg_twin.assign(d->seg_twin, d->seg_twin + d->n_seg);
    h->seg_normal.assign(d->seg_normal, d->seg_normal + 2 * d->n_seg);
  }
  h->d.sub_point_offset = h->sub_off.data();
  h->d.sub_n_res = h->n_res.data();
  h->d.sub_n_data = h->n_data.data();
  h->d.sub_seg_offset = h->seg_off.data();
  h->d.sub_hparams = h->hp.data();
  h->d.seg_n = h->seg_n.data();
  h->d.seg_twin = h->seg_twin.data();
  h->d.seg_normal = h->seg_normal.data();
  h->d.sub_norm_counts = d->sub_norm_counts ? h->norm_counts.data() : nullptr;
  if (d->sub_activation)
    h->act.assign(d->sub_activation, d->sub_activation + ns);
  else
    h->act.assign(ns, d->activation);
  h->d.sub_activation = h->act.data();
  if (d->n_peers > 0) {
    h->peer_rank.assign(d->peer_rank, d->peer_rank + d->n_peers);
    h->peer_send_off.assign(d->peer_send_off, d->peer_send_off + d->n_peers + 1);
    h->send_rows.assign(d->send_rows, d->send_rows + h->peer_send_off.back());
    h->peer_recv_row.assign(d->peer_recv_row, d->peer_recv_row + d->n_peers);
    h->peer_recv_n.assign(d->peer_recv_n, d->peer_recv_n + d->n_peers);
  }
  h->d.peer_rank = h->peer_rank.data();
  h->d.peer_send_off = h->peer_send_off.data();
  h->d.send_rows = h->send_rows.data();
  h->d.peer_recv_row = h->peer_recv_row.data();
  h->d.peer_recv_n = h->peer_recv_n.data();
  h->d.nccl_id = nullptr;   // consumed below (the communicator is the handle's)
  if (d->geometry != PINN_DD_GEOM_NONE) {
    h->geo.assign(d->geo, d->geo + size_t(d->n_geo) * (d->geometry == PINN_DD_GEOM_BOXES ? 4 : 2));
    h->geo_local.assign(d->geo_local, d->geo_local + d->n_geo);
    if (d->geometry == PINN_DD_GEOM_VORONOI) h->poly.assign(d->poly, d->poly + 2 * size_t(d->n_poly));
  }
  h->d.geo = h->geo.data();
  h->d.geo_local = h->geo_local.data();
  h->d.poly = h->poly.data();
  h->stream = static_cast<cudaStream_t>(d->stream);

  char* base = static_cast<char*>(ws);
  h->params = reinterpret_cast<float*>(base + L.params);
  h->m = reinterpret_cast<float*>(base + L.m);
  h->v = reinterpret_cast<float*>(base + L.v);
  h->grad = reinterpret_cast<float*>(base + L.grad);
  h->scratch = reinterpret_cast<float*>(base + L.scratch);
  h->partial = reinterpret_cast<float*>(base + L.partial);
  h->partial_loss = reinterpret_cast<float*>(base + L.ploss);
  h->payload = reinterpret_cast<float*>(base + L.payload);
  h->pinfo = reinterpret_cast<int32_t*>(base + L.pinfo);
  h->pinv = reinterpret_cast<float*>(base + L.pinv);
  h->ptwin = reinterpret_cast<int32_t*>(base + L.ptwin);
  h->segn = reinterpret_cast<float2*>(base + L.segn);
  h->sub_w = reinterpret_cast<float4*>(base + L.subw);
  h->sub_act = reinterpret_cast<int32_t*>(base + L.subact);
  h->sub_adam = reinterpret_cast<float4*>(base + L.suba);
  h->chunks1 = reinterpret_cast<Chunk*>(base + L.ch1);
  h->order1 = reinterpret_cast<int32_t*>(base + L.ord1);
  h->sched = reinterpret_cast<int32_t*>(base + L.sched);
  h->chunks2 = reinterpret_cast<Chunk*>(base + L.ch2);
  h->sub_chunk = reinterpret_cast<int32_t*>(base + L.subch);
  h->tstep = reinterpret_cast<int32_t*>(base + L.tstep);
  h->done = reinterpret_cast<int32_t*>(base + L.done);
  h->sflag = reinterpret_cast<int32_t*>(base + L.sflag);
  h->slope_part = reinterpret_cast<double*>(base + L.slopep);
  h->loss = reinterpret_cast<float*>(base + L.loss);
  h->packmap = reinterpret_cast<int32_t*>(base + L.packmap);
  h->gstash = reinterpret_cast<float*>(base + L.gstash);
  h->sendbuf = reinterpret_cast<float*>(base + L.sendbuf);
  h->psend = reinterpret_cast<int32_t*>(base + L.psend);
  h->dgeo = reinterpret_cast<float*>(base + L.dgeo);
  h->dpoly = reinterpret_cast<float*>(base + L.dpoly);
  h->dgeo_local = reinterpret_cast<int32_t*>(base + L.dgeoloc);
  h->xflags = reinterpret_cast<unsigned long long*>(base + L.xflags);
  h->xstep = reinterpret_cast<int*>(base + L.xstep);
  h->sub_ctr = reinterpret_cast<int32_t*>(base + L.sctr);
  h->sub_tiles = reinterpret_cast<int32_t*>(base + L.stiles);

  // ---- per-point classification and 1/N (Eq. 3/5/6; per-edge mean, Z2)
  const int64_t np = d->n_points;
  std::vector<int32_t> pinfo(np + 1, 0), ptwin(np + 1, 0);
  std::vector<float> pinv(np + 1, 0.0f);
  for (int q = 0; q < ns; ++q) {
    const int64_t off = h->sub_off[q];
    const int nr = h->n_res[q], nd = h->n_data[q];
    // 1/N of MSE_F and MSE_u: local counts, or the full-data counts of a shard
    const int cr = h->norm_counts.empty() ? nr : h->norm_counts[2 * q];
    const int cd = h->norm_counts.empty() ? nd : h->norm_counts[2 * q + 1];
    for (int64_t p = off; p < off + nr; ++p) {
      pinfo[p] = 0;
      pinv[p] = 1.0f / float(cr);
    }
    for (int64_t p = off + nr; p < off + nr + nd; ++p) {
      pinfo[p] = 1;
      pinv[p] = 1.0f / float(cd);
    }
    int64_t p = off + nr + nd;
    for (int sgi = h->seg_off[q]; sgi < h->seg_off[q + 1]; ++sgi) {
      const int n = h->seg_n[sgi];
      // interface condition of this edge: flux (cPINN, or HYBRID on an x1-normal
      // edge) or residual (XPINN, or HYBRID on an x2-normal edge)
      const bool flux = d->method == PINN_DD_METHOD_CPINN ||
                        (d->method == PINN_DD_METHOD_HYBRID && h->seg_normal[2 * sgi + 1] == 0.0f);
      for (int j = 0; j < n; ++j, ++p) {
        pinfo[p] = 2 | (flux ? 4 : 0) | (sgi << 3);
        pinv[p] = 1.0f / float(n);
        ptwin[p] = int32_t(h->seg_twin[sgi] + j);
      }
    }
  }
  // a local twin must be the first point of another segment of the same
  // edge: same N_I, same interface condition, same canonical normal (Z3)
  {
    std::vector<int64_t> seg_start(d->n_seg);
    for (int q = 0; q < ns; ++q) {
      int64_t p0 = h->sub_off[q] + h->n_res[q] + h->n_data[q];
      for (int sgi = h->seg_off[q]; sgi < h->seg_off[q + 1]; ++sgi) {
        seg_start[sgi] = p0;
        p0 += h->seg_n[sgi];
      }
    }
    for (int sgi = 0; sgi < d->n_seg; ++sgi) {
      const int64_t tw = h->seg_twin[sgi];
      if (tw >= np) continue;   // received rows: validated by the sender's plan
      const int32_t info = pinfo[tw];
      const int ts = (info & 3) == 2 ? (info >> 3) : -1;
      const char* why = nullptr;
      if (ts < 0 || seg_start[ts] != tw) why = "is not the first point of an interface segment";
      else if (ts == sgi) why = "is the segment itself";
      else if (h->seg_n[ts] != h->seg_n[sgi]) why = "belongs to a segment with a different N_I";
      else if ((pinfo[tw] & 4) != (pinfo[seg_start[sgi]] & 4)) why = "belongs to a segment with another condition";
      else if (h->seg_normal[2 * ts] != h->seg_normal[2 * sgi] || h->seg_normal[2 * ts + 1] != h->seg_normal[2 * sgi + 1])
        why = "belongs to a segment with another normal";
      if (why) {
        s = fail(nullptr, PINN_DD_EPROTOCOL, "segment %d: twin row %lld %s", sgi, (long long)tw, why);
        delete h;
        return s;
      }
    }
  }
  // send slot of every point of a cut edge (K2 writes its payload row there too)
  std::vector<int32_t> psend(np + 1, -1);
  for (size_t j = 0; j < h->send_rows.size(); ++j) {
    const int64_t r = h->send_rows[j];
    if ((pinfo[r] & 3) != 2 || psend[r] != -1) {
      s = fail(nullptr, PINN_DD_EPROTOCOL, "send row %lld is not an interface point or is sent twice", (long long)r);
      delete h;
      return s;
    }
    psend[r] = int32_t(j);
  }
  std::vector<float4> subw(ns), suba(ns);
  for (int q = 0; q < ns; ++q) {
    subw[q] = make_float4(h->hp[q].w_u, h->hp[q].w_f, h->hp[q].w_i, h->hp[q].w_if);
    suba[q] = make_float4(h->hp[q].lr, h->hp[q].beta1, h->hp[q].beta2, h->hp[q].eps);
  }
  // ---- chunks: K1 over all points, K2 over interface points
  const int P = h->ops->P;
  std::vector<Chunk> c1, c2;
  std::vector<int32_t> subch(ns + 1, 0);
  for (int q = 0; q < ns; ++q) {
    subch[q] = int32_t(c1.size());
    const int off = h->sub_off[q], cnt = h->sub_off[q + 1] - off;
    const int na = h->n_res[q] + h->n_data[q];
    int s0 = 0;
    for (int sz : split_chunks(na, cnt - na, P, h->ops->pstride)) {
      const bool iface = sz < 0;
      if (iface) sz = -sz - 1;
      c1.push_back(Chunk{q, off + s0, sz, iface ? 1 : 0});
      s0 += sz;
    }
    const int i0 = off + h->n_res[q] + h->n_data[q];
    const int ni = h->sub_off[q + 1] - i0;
    for (int s0 = 0; s0 < ni; s0 += P) c2.push_back(Chunk{q, i0 + s0, std::min(P, ni - s0), 0});
  }
  subch[ns] = int32_t(c1.size());
  // K1 processing orders, larger chunks first (stable), the one-tile tail last:
  // [0, n1) every chunk (pinn_dd_loss_grad); [n1, n1 + n_int) residual/training
  // chunks, then [n1 + n_int, 2 n1) interface chunks (the phased calls)
  std::vector<int32_t> ord1(2 * c1.size());
  auto big_first = [&](int32_t x, int32_t y) { return c1[x].count > c1[y].count; };
  for (size_t i = 0; i < c1.size(); ++i) ord1[i] = int32_t(i);
  std::stable_sort(ord1.begin(), ord1.begin() + c1.size(), big_first);
  int n_int = 0;
  for (size_t i = 0; i < c1.size(); ++i)
    if (!c1[i].pad) ord1[c1.size() + n_int++] = int32_t(i);
  int k = n_int;
  for (size_t i = 0; i < c1.size(); ++i)
    if (c1[i].pad) ord1[c1.size() + k++] = int32_t(i);
  std::stable_sort(ord1.begin() + c1.size(), ord1.begin() + c1.size() + n_int, big_first);
  std::stable_sort(ord1.begin() + c1.size() + n_int, ord1.end(), big_first);
  h->n_int = n_int;
  // per-subdomain queues of the fused step: a subdomain's chunks in chunk
  // order, which split_chunks makes residual + training chunks largest first,
  // then interface chunks largest first (checked here; else no sticky queues);
  // cumulative tiles place the CTAs' first claims
  std::vector<int32_t> stiles(ns + 1, 0);
  h->sticky_order = true;
  for (int q = 0; q < ns; ++q) {
    int tiles = 0;
    for (int32_t i = subch[q]; i < subch[q + 1]; ++i) {
      tiles += (c1[i].count + P - 1) / P;
      if (i > subch[q]) {
        const Chunk &u = c1[i - 1], &v = c1[i];
        if (u.pad > v.pad || (u.pad == v.pad && u.count < v.count)) h->sticky_order = false;
      }
    }
    stiles[q + 1] = stiles[q] + tiles;
  }
  h->sub_list_tiles = stiles[ns];
  std::vector<int32_t> pm;
  h->ops->packmap(pm);
  h->n_packed = int(pm.size());

  cudaStream_t st = h->stream;
#define CKC(call)                                                                                  \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      fail(nullptr, PINN_DD_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));                       \
      delete h;                                                                                    \
      return PINN_DD_ECUDA;                                                                        \
    }                                                                                              \
  } while (0)
  CKC(h->ops->setattr(h->ops->smem));
  const size_t pbytes = size_t(ns) * h->pstride * sizeof(float);
  CKC(cudaMemsetAsync(h->params, 0, pbytes, st));
  CKC(cudaMemsetAsync(h->m, 0, pbytes, st));
  CKC(cudaMemsetAsync(h->v, 0, pbytes, st));
  CKC(cudaMemsetAsync(h->grad, 0, pbytes, st));
  {
    const size_t nslots = (d->flags & PINN_DD_FLAG_PEER_STORES) ? 2 : 1;
    CKC(cudaMemsetAsync(h->payload, 0, (size_t(np) + nslots * d->n_recv + 1) * h->nf * sizeof(float), st));
  }
  CKC(cudaMemsetAsync(h->xflags, 0, kMaxPeers * sizeof(unsigned long long), st));
  CKC(cudaMemsetAsync(h->xstep, 0, sizeof(int), st));
  // K1 never writes a partial's padding slots; K5a sums every index, so they start (and stay) 0
  CKC(cudaMemsetAsync(h->partial, 0, size_t(h->n_chunks1) * h->pstride * sizeof(float), st));
  CKC(cudaMemcpyAsync(h->pinfo, pinfo.data(), pinfo.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->pinv, pinv.data(), pinv.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->ptwin, ptwin.data(), ptwin.size() * 4, cudaMemcpyHostToDevice, st));
  if (d->n_seg > 0)
    CKC(cudaMemcpyAsync(h->segn, h->seg_normal.data(), h->seg_normal.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->sub_w, subw.data(), subw.size() * sizeof(float4), cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->sub_act, h->act.data(), h->act.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->sub_adam, suba.data(), suba.size() * sizeof(float4), cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->chunks1, c1.data(), c1.size() * sizeof(Chunk), cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->order1, ord1.data(), ord1.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->sub_tiles, stiles.data(), stiles.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemsetAsync(h->sub_ctr, 0, ns * 4, st));
  CKC(cudaMemsetAsync(h->sched, 0, 8 * sizeof(int32_t), st));
  if (!c2.empty())
    CKC(cudaMemcpyAsync(h->chunks2, c2.data(), c2.size() * sizeof(Chunk), cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->sub_chunk, subch.data(), subch.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemsetAsync(h->tstep, 0, ns * 4, st));
  CKC(cudaMemsetAsync(h->done, 0, ns * 4, st));
  CKC(cudaMemsetAsync(h->sflag, 0, ns * 4, st));
  CKC(cudaMemsetAsync(h->loss, 0, ns * 8 * 4, st));
  CKC(cudaMemcpyAsync(h->packmap, pm.data(), pm.size() * 4, cudaMemcpyHostToDevice, st));
  CKC(cudaMemcpyAsync(h->psend, psend.data(), psend.size() * 4, cudaMemcpyHostToDevice, st));
  if (!h->geo.empty()) {
    CKC(cudaMemcpyAsync(h->dgeo, h->geo.data(), h->geo.size() * 4, cudaMemcpyHostToDevice, st));
    CKC(cudaMemcpyAsync(h->dgeo_local, h->geo_local.data(), h->geo_local.size() * 4, cudaMemcpyHostToDevice, st));
  }
  if (!h->poly.empty()) CKC(cudaMemcpyAsync(h->dpoly, h->poly.data(), h->poly.size() * 4, cudaMemcpyHostToDevice, st));
  {
    // initial parameters: the caller's, or W = b = 0 with a^k = 1/n (Z6).  The
    // slope gradient comes from a^k dJ/da^k = <W, dJ/dW> + <b, dJ/db> (DESIGN.md
    // 5.3), which needs a^k != 0: a zero slope is rejected here.
    std::vector<float> init(size_t(ns) * h->n_packed, 0.0f);
    std::vector<int> slot_a;
    for (int k = 0, o = 0; k < d->n_hidden; ++k) {
      o += (k == 0 ? 2 : d->width) * d->width + d->width;
      slot_a.push_back(o);
      o += 1;
    }
    if (d->init_params) {
      CKC(cudaMemcpyAsync(init.data(), d->init_params, init.size() * 4, cudaMemcpyDeviceToHost, st));
      CKC(cudaStreamSynchronize(st));
      for (int q = 0; q < ns; ++q)
        for (int k = 0; k < d->n_hidden; ++k)
          if (!(std::isfinite(init[size_t(q) * h->n_packed + slot_a[k]]) &&
                init[size_t(q) * h->n_packed + slot_a[k]] != 0.0f)) {
            fail(nullptr, PINN_DD_EINVAL, "subdomain %d: slope a^%d = %g must be finite and non-zero", q, k + 1,
                 double(init[size_t(q) * h->n_packed + slot_a[k]]));
            delete h;
            return PINN_DD_EINVAL;
          }
    } else {
      for (int q = 0; q < ns; ++q)
        for (int k = 0; k < d->n_hidden; ++k) init[size_t(q) * h->n_packed + slot_a[k]] = 1.0f / d->slope_n;
    }
    CKC(cudaMemcpyAsync(h->scratch, init.data(), init.size() * 4, cudaMemcpyHostToDevice, st));
    dim3 g((h->n_packed + 255) / 256, ns);
    k_scatter<<<g, 256, 0, st>>>(h->scratch, h->packmap, h->n_packed, h->pstride, h->n_packed, h->params, ns);
    CKC(cudaGetLastError());
    CKC(cudaStreamSynchronize(st));   // `init` goes out of scope
  }
  for (auto& e : h->ev) CKC(cudaEventCreate(&e));
  for (auto& e : h->gjoin) CKC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CKC(cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking));
  CKC(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
  CKC(cudaEventCreateWithFlags(&h->xfork, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&h->xjoin, cudaEventDisableTiming));
  if (d->nccl_id) {
    // join the exchange communicator (collective over the `world` ranks)
    const Nccl& N = nccl();
    if (!N.ok) {
      fail(nullptr, PINN_DD_ENCCL, "NCCL transport requested but unavailable: %s", N.why.c_str());
      pinn_dd_destroy(h);
      return PINN_DD_ENCCL;
    }
    ncclUniqueId id;
    std::memcpy(&id, d->nccl_id, sizeof id);
    const ncclResult_t r = N.CommInitRank(&h->comm, d->world, id, d->rank);
    if (r != 0) {
      h->comm = nullptr;
      fail(nullptr, PINN_DD_ENCCL, "ncclCommInitRank(world %d, rank %d): %s", d->world, d->rank,
           N.GetErrorString(r));
      pinn_dd_destroy(h);
      return PINN_DD_ENCCL;
    }
  }
  CKC(cudaStreamSynchronize(st));   // host vectors above go out of scope
  *out = h;
  return PINN_DD_OK;
}

// per-call timing of the phased entry points (PINN_DD_FLAG_TIMING): events 4/5
static pinn_dd_status phase_begin(pinn_dd* h) {
  if (h->d.flags & PINN_DD_FLAG_TIMING) CK(h, cudaEventRecord(h->ev[7], h->stream));
  return PINN_DD_OK;
}
static pinn_dd_status phase_end(pinn_dd* h, int slot, int slot2 = -1) {
  if (h->d.flags & PINN_DD_FLAG_TIMING) {
    CK(h, cudaEventRecord(h->ev[8], h->stream));
    CK(h, cudaEventSynchronize(h->ev[8]));
    float ms = 0;
    CK(h, cudaEventElapsedTime(&ms, h->ev[7], h->ev[8]));
    h->ms[slot] += ms;
    if (slot2 >= 0) h->ms[slot2] += ms;
  }
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_interface_payload(pinn_dd* h) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  pinn_dd_status s;
  if ((s = phase_begin(h)) != PINN_DD_OK || (s = launch_k2(h)) != PINN_DD_OK) return s;
  return phase_end(h, 0);
}

pinn_dd_status pinn_dd_payload_buffer(pinn_dd* h, float** buf, int32_t* n_fields, int64_t* n_rows) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  if (buf) *buf = h->payload;
  if (n_fields) *n_fields = h->nf;
  if (n_rows) *n_rows = h->d.n_points + h->d.n_recv;
  return PINN_DD_OK;
}

// K5a (reduce + slopes) and the optional copies of pinn_dd_loss_grad
static pinn_dd_status finish_loss_grad(pinn_dd* h, float* loss_dev, float* grad_dev) {
  pinn_dd_status s;
  if ((s = phase_begin(h)) != PINN_DD_OK || (s = launch_k5(h, 0)) != PINN_DD_OK || (s = phase_end(h, 2)) != PINN_DD_OK)
    return s;
  if (loss_dev)
    CK(h, cudaMemcpyAsync(loss_dev, h->loss, size_t(h->d.n_sub) * 8 * 4, cudaMemcpyDeviceToDevice, h->stream));
  if (grad_dev) {
    dim3 g((h->n_packed + 255) / 256, h->d.n_sub);
    k_gather<<<g, 256, 0, h->stream>>>(h->grad, h->packmap, h->n_packed, h->pstride, h->n_packed, grad_dev,
                                       h->d.n_sub);
    CK(h, cudaGetLastError());
  }
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_loss_grad(pinn_dd* h, float* loss_dev, float* grad_dev) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  pinn_dd_status s;
  if ((s = phase_begin(h)) != PINN_DD_OK || (s = launch_k1(h)) != PINN_DD_OK || (s = phase_end(h, 1)) != PINN_DD_OK)
    return s;
  return finish_loss_grad(h, loss_dev, grad_dev);
}

pinn_dd_status pinn_dd_loss_grad_interior(pinn_dd* h) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  pinn_dd_status s;
  if ((s = phase_begin(h)) != PINN_DD_OK || (s = launch_k1(h, 1)) != PINN_DD_OK) return s;
  return phase_end(h, 1, 5);
}

pinn_dd_status pinn_dd_loss_grad_interface(pinn_dd* h, float* loss_dev, float* grad_dev) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  pinn_dd_status s;
  if ((s = phase_begin(h)) != PINN_DD_OK || (s = launch_k1(h, 2)) != PINN_DD_OK || (s = phase_end(h, 1, 6)) != PINN_DD_OK)
    return s;
  return finish_loss_grad(h, loss_dev, grad_dev);
}

pinn_dd_status pinn_dd_adam(pinn_dd* h) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  pinn_dd_status s;
  if ((s = phase_begin(h)) != PINN_DD_OK || (s = launch_k5(h, 2)) != PINN_DD_OK) return s;
  return phase_end(h, 2);
}

pinn_dd_status pinn_dd_step(pinn_dd* h, int32_t n_iters, float* loss_host) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  if (remote(h) && !h->comm)
    return fail(h, PINN_DD_EPROTOCOL,
                "pinn_dd_step with remote twins (n_recv = %lld) needs a transport: NCCL (desc nccl_id) or "
                "connected peer stores (PINN_DD_FLAG_PEER_STORES + pinn_dd_connect_peers); else use the "
                "phased calls",
                (long long)h->d.n_recv);
  if (n_iters < 0) return fail(h, PINN_DD_EINVAL, "n_iters < 0");
  const bool timed = (h->d.flags & PINN_DD_FLAG_TIMING) != 0;
  const bool graph = (h->d.flags & PINN_DD_FLAG_GRAPH) != 0;
  pinn_dd_status s;
  for (int it = 0; it < n_iters; ++it) {
    if (graph) {
      if (!h->gexec) {
        cudaGraph_t g;
        if (remote(h)) {
          // NCCL connects peers lazily on the first send / receive (allocations,
          // IPC mappings): one eager exchange before capture (every rank calls
          // pinn_dd_step, so the peers take part; the rows it moves are
          // rewritten by K2 before they are read)
          if ((s = nccl_group(h, h->stream)) != PINN_DD_OK) return s;
          CK(h, cudaStreamSynchronize(h->stream));
        }
        const long long before = h->launches;
        cudaStream_t user = h->stream;
        h->stream = h->gstream;
        cudaError_t e0 = cudaStreamBeginCapture(
            h->stream, remote(h) ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeThreadLocal);
        if (e0 != cudaSuccess) {
          h->stream = user;
          return fail(h, PINN_DD_ECUDA, "graph capture: %s", cudaGetErrorString(e0));
        }
        pinn_dd_status cs = one_iteration(h, timed, true);
        cudaError_t e = cudaStreamEndCapture(h->stream, &g);
        h->stream = user;
        if (cs != PINN_DD_OK) return cs;
        if (e != cudaSuccess) return fail(h, PINN_DD_ECUDA, "graph capture: %s", cudaGetErrorString(e));
        CK(h, cudaGraphInstantiate(&h->gexec, g, 0));
        cudaGraphDestroy(g);
        h->launches = before;   // counted on every replay below
      }
      CK(h, cudaEventRecord(h->gjoin[0], h->stream));
      CK(h, cudaStreamWaitEvent(h->gstream, h->gjoin[0], 0));
      CK(h, cudaGraphLaunch(h->gexec, h->gstream));
      CK(h, cudaEventRecord(h->gjoin[1], h->gstream));
      CK(h, cudaStreamWaitEvent(h->stream, h->gjoin[1], 0));
      h->launches += iteration_launches(h);
      if (timed && (s = accumulate_times(h, timing_kind(h))) != PINN_DD_OK) return s;
    } else if ((s = one_iteration(h, timed, false)) != PINN_DD_OK) {
      return s;
    }
  }
  if (loss_host) {
    CK(h, cudaMemcpyAsync(loss_host, h->loss, size_t(h->d.n_sub) * 8 * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return check_status(h, loss_host);
  }
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_predict(pinn_dd* h, const float* pts, int64_t n, float* out, int32_t mode) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  if (n < 0 || (n > 0 && (!pts || !out))) return fail(h, PINN_DD_EINVAL, "bad predict arguments");
  if (mode != PINN_DD_PREDICT_STITCHED && mode != PINN_DD_PREDICT_OWNER)
    return fail(h, PINN_DD_EINVAL, "bad predict mode %d", mode);
  if (h->d.geometry == PINN_DD_GEOM_NONE)
    return fail(h, PINN_DD_EINVAL, "pinn_dd_predict needs desc geometry (or use pinn_dd_predict_owners)");
  Geo g{h->d.geometry, mode, nullptr, h->d.n_geo, h->dgeo, h->dgeo_local, int(h->poly.size() / 2), h->dpoly,
        h->d.geo_tol};
  h->ops->pred(h->params, h->pstride, h->d.slope_n, pts, g, n, out, h->sub_act, h->stream);
  ++h->launches;
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_predict_owners(pinn_dd* h, const float* pts, const int32_t* owners, int64_t n, float* out) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  if (n < 0 || (n > 0 && (!pts || !owners || !out))) return fail(h, PINN_DD_EINVAL, "bad predict arguments");
  Geo g{0, 0, owners, 0, nullptr, nullptr, 0, nullptr, 0.0f};
  h->ops->pred(h->params, h->pstride, h->d.slope_n, pts, g, n, out, h->sub_act, h->stream);
  ++h->launches;
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}

static float* state_ptr(pinn_dd* h, int what) {
  switch (what) {
    case 0: return h->params;
    case 1: return h->m;
    case 2: return h->v;
    case 3: return h->grad;
    default: return nullptr;
  }
}

pinn_dd_status pinn_dd_get_params(pinn_dd* h, int32_t sub, int32_t what, float* dst) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  float* src = state_ptr(h, what);
  if (!src || sub < 0 || sub >= h->d.n_sub || !dst) return fail(h, PINN_DD_EINVAL, "bad get_params arguments");
  dim3 g((h->n_packed + 255) / 256, 1);
  k_gather<<<g, 256, 0, h->stream>>>(src + size_t(sub) * h->pstride, h->packmap, h->n_packed, h->pstride,
                                     h->n_packed, dst, 1);
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_set_params(pinn_dd* h, int32_t sub, int32_t what, const float* src) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  float* dst = state_ptr(h, what);
  if (!dst || sub < 0 || sub >= h->d.n_sub || !src) return fail(h, PINN_DD_EINVAL, "bad set_params arguments");
  dim3 g((h->n_packed + 255) / 256, 1);
  k_scatter<<<g, 256, 0, h->stream>>>(src, h->packmap, h->n_packed, h->pstride, h->n_packed,
                                      dst + size_t(sub) * h->pstride, 1);
  CK(h, cudaGetLastError());
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_get_step(pinn_dd* h, int32_t sub, int32_t* t) {
  if (!h || !t || sub < 0 || sub >= h->d.n_sub) return fail(h, PINN_DD_EINVAL, "bad get_step arguments");
  CK(h, cudaMemcpyAsync(t, h->tstep + sub, 4, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_kernel_times(pinn_dd* h, double* ms8) {
  if (!h || !ms8) return fail(h, PINN_DD_EINVAL, "bad kernel_times arguments");
  CK(h, cudaStreamSynchronize(h->stream));
  for (int i = 0; i < 8; ++i) ms8[i] = h->ms[i];
  ms8[3] = double(h->launches);
  for (double& v : h->ms) v = 0.0;
  h->launches = 0;
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_exchange(pinn_dd* h) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  if (!remote(h)) return PINN_DD_OK;
  if (!h->comm) return fail(h, PINN_DD_EPROTOCOL, "pinn_dd_exchange needs the NCCL transport (desc nccl_id)");
  return nccl_group(h, h->stream);
}

pinn_dd_status pinn_dd_ipc_export(pinn_dd* h, void* handle64, int64_t* flags_offset, int64_t* rows_offset) {
  if (!h || !handle64 || !flags_offset || !rows_offset) return fail(h, PINN_DD_EINVAL, "bad ipc_export arguments");
  if (!(h->d.flags & PINN_DD_FLAG_PEER_STORES)) return fail(h, PINN_DD_EINVAL, "handle without PINN_DD_FLAG_PEER_STORES");
  cudaIpcMemHandle_t ih;
  CK(h, cudaIpcGetMemHandle(&ih, h->payload));
  // offsets inside the allocation the handle maps: its base via the driver API
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = [] {
    void* lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libcuda.so.1", RTLD_NOW);
    return lib ? reinterpret_cast<GetRange>(dlsym(lib, "cuMemGetAddressRange_v2")) : nullptr;
  }();
  if (!get_range) return fail(h, PINN_DD_ECUDA, "cuMemGetAddressRange_v2 unavailable");
  unsigned long long b = 0;
  size_t sz = 0;
  if (get_range(&b, &sz, reinterpret_cast<unsigned long long>(h->payload)) != 0)
    return fail(h, PINN_DD_ECUDA, "cuMemGetAddressRange_v2 failed");
  std::memcpy(handle64, &ih, sizeof ih);
  *flags_offset = int64_t(reinterpret_cast<uintptr_t>(h->xflags) - b);
  *rows_offset = int64_t(reinterpret_cast<uintptr_t>(h->payload) - b);
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_connect_peers(pinn_dd* h, const void* handles, const int64_t* flags_offset,
                                     const int64_t* rows_offset, const int64_t* peer_row, const int64_t* peer_nrecv,
                                     const int32_t* peer_flag) {
  if (!h) return fail(nullptr, PINN_DD_EINVAL, "handle is NULL");
  if (!(h->d.flags & PINN_DD_FLAG_PEER_STORES)) return fail(h, PINN_DD_EINVAL, "handle without PINN_DD_FLAG_PEER_STORES");
  const int n = int(h->peer_rank.size());
  if (n == 0) return PINN_DD_OK;
  if (!handles || !flags_offset || !rows_offset || !peer_row || !peer_nrecv || !peer_flag)
    return fail(h, PINN_DD_EINVAL, "bad connect_peers arguments");
  if (h->ops->kf == nullptr || h->n_chunks2 == 0)
    return fail(h, PINN_DD_EUNSUPPORTED, "peer stores need the fused step (interface points on this handle)");
  PeerX px{};
  px.n = n;
  for (int i = 0; i <= n; ++i) px.send_off[i] = h->peer_send_off[i];
  for (int i = 0; i < n; ++i) {
    char* base;
    if (h->peer_rank[i] == h->d.rank) {
      base = nullptr;   // loop-back: this handle's own region
    } else {
      cudaIpcMemHandle_t ih;
      std::memcpy(&ih, static_cast<const char*>(handles) + 64 * size_t(i), sizeof ih);
      void* p = nullptr;
      CK(h, cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
      h->ipc_open.push_back(p);
      base = static_cast<char*>(p);
    }
    float* rows = base ? reinterpret_cast<float*>(base + rows_offset[i]) : h->payload;
    unsigned long long* flags = base ? reinterpret_cast<unsigned long long*>(base + flags_offset[i]) : h->xflags;
    if (peer_flag[i] < 0 || peer_flag[i] >= kMaxPeers || peer_nrecv[i] < 0 || peer_row[i] < 0)
      return fail(h, PINN_DD_EPROTOCOL, "peer %d: bad row / flag description", i);
    px.dst[i] = rows + size_t(peer_row[i]) * h->nf;
    px.slot_stride[i] = peer_nrecv[i] * h->nf;
    px.peer_flag[i] = flags + peer_flag[i];
    px.expect[i] = h->peer_recv_n[i];
  }
  px.my_flag = h->xflags;
  px.n_recv = h->d.n_recv;
  px.step = h->xstep;
  h->px = px;
  h->peers_connected = true;
  if (h->gexec) {   // the captured step graph predates the transport
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_nccl_unique_id(void* id128) {
  if (!id128) return fail(nullptr, PINN_DD_EINVAL, "id128 is NULL");
  const Nccl& N = nccl();
  if (!N.ok) return fail(nullptr, PINN_DD_ENCCL, "NCCL unavailable: %s", N.why.c_str());
  ncclUniqueId id;
  const ncclResult_t r = N.GetUniqueId(&id);
  if (r != 0) return fail(nullptr, PINN_DD_ENCCL, "ncclGetUniqueId: %s", N.GetErrorString(r));
  std::memcpy(id128, &id, sizeof id);
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_read_loss(pinn_dd* h, float* dst) {
  if (!h || !dst) return fail(h, PINN_DD_EINVAL, "bad read_loss arguments");
  CK(h, cudaMemcpyAsync(dst, h->loss, size_t(h->d.n_sub) * 8 * 4, cudaMemcpyDefault, h->stream));
  return PINN_DD_OK;
}

int32_t pinn_dd_step_fused(const pinn_dd* h) { return h && use_fused(h) ? 1 : 0; }

pinn_dd_status pinn_dd_plan_info(pinn_dd* h, int64_t* info4) {
  if (!h || !info4) return fail(h, PINN_DD_EINVAL, "bad plan_info arguments");
  info4[0] = h->ops->P;
  info4[1] = h->tpc;
  info4[2] = h->n_chunks1;
  info4[3] = h->grid1;
  return PINN_DD_OK;
}

pinn_dd_status pinn_dd_debug_buffer(pinn_dd* h, int32_t which, void** ptr, int64_t* bytes) {
  if (!h || !ptr || !bytes) return fail(h, PINN_DD_EINVAL, "bad debug_buffer arguments");
  const int64_t np = h->d.n_points + 1, ns = h->d.n_sub;
  switch (which) {
    case 0: *ptr = h->pinfo; *bytes = np * 4; break;
    case 1: *ptr = h->pinv; *bytes = np * 4; break;
    case 2: *ptr = h->ptwin; *bytes = np * 4; break;
    case 3: *ptr = h->chunks1; *bytes = int64_t(h->n_chunks1) * sizeof(Chunk); break;
    case 4: *ptr = h->chunks2; *bytes = int64_t(h->n_chunks2) * sizeof(Chunk); break;
    case 5: *ptr = h->partial; *bytes = int64_t(h->n_chunks1) * h->pstride * 4; break;
    case 6: *ptr = h->params; *bytes = ns * h->pstride * 4; break;
    default: return fail(h, PINN_DD_EINVAL, "unknown debug buffer %d", which);
  }
  return PINN_DD_OK;
}

void pinn_dd_destroy(pinn_dd* h) {
  if (!h) return;
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->gjoin)
    if (e) cudaEventDestroy(e);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->comm) nccl().CommDestroy(h->comm);
  for (void* p : h->ipc_open) cudaIpcCloseMemHandle(p);
  if (h->cstream) cudaStreamDestroy(h->cstream);
  if (h->xfork) cudaEventDestroy(h->xfork);
  if (h->xjoin) cudaEventDestroy(h->xjoin);
  delete h;
}

const char* pinn_dd_last_error(const pinn_dd* h) {
  if (!h) return g_create_error.c_str();
  return h->err.c_str();
}

}  // extern "C"
