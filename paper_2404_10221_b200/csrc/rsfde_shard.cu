// Slab-sharded 3D solver: the grid is split along x1 over P ranks (x1 padded to
// n1+1 so every rank owns s = (n1+1)/P planes; the pad plane is the DST-I zero).  One GMRES
// iteration K v = P_hat^{-1} A v runs as
//   [x1-slabs, layout A = [x1 local][x2][x3 (+pad)]]  spectral operator passes along x3 and x2
//   all-to-all transpose of the two pass outputs to x2-slabs, layout T = [x2 local][x3][x1 (+pad)]
//   [layout T]  the last operator pass along x1 with DST . Lambda_hat^{-1} . DST fused
//   all-to-all transpose back, inverse DSTs along x2 and x3 in layout A
// i.e. three vector transposes per iteration; the CGS2 dot products and norms are reduced over
// the ranks (allreduce).  The transport is NCCL (one rank per process, ncclSend/ncclRecv groups
// and ncclAllReduce, libnccl.so.2 loaded with dlopen) or, with all P ranks in one process
// (nlocal == P), device copies -- the single-GPU emulation used by the parity tests.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx_internal.h"

using namespace rsfde;

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
      nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    Send = (decltype(Send))dlsym(h, "ncclSend");
    Recv = (decltype(Recv))dlsym(h, "ncclRecv");
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    ErrStr = (decltype(ErrStr))dlsym(h, "ncclGetErrorString");
    return CommInitRank && CommDestroy && GetUniqueId && Send && Recv && GroupStart && GroupEnd && AllReduce;
  }
};
NcclApi g_nccl;
thread_local std::string g_team_error;


// ------------------------------------------------------------------------------ transposes
// A = [x1l < s][x2 < n2][x3 < P3]  ->  send block r' (x2 in [r' s2, (r'+1) s2)) = [x2l][x3 < n3][x1l < s]
__global__ void pack_AT_kernel(const double* __restrict__ A, double* __restrict__ send, int s, int n2, int n3,
                               int P3, int s2, long long blk) {
  __shared__ double tile[32][33];
  const int x2 = blockIdx.z;
  const int x3_0 = blockIdx.x * 32, x1_0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int x1l = x1_0 + i, x3 = x3_0 + threadIdx.x;
    tile[i][threadIdx.x] = (x1l < s && x3 < n3 && x2 < n2) ? A[((long long)x1l * n2 + x2) * P3 + x3] : 0.0;
  }
  __syncthreads();
  const int rp = x2 / s2, x2l = x2 % s2;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int x3 = x3_0 + i, x1l = x1_0 + threadIdx.x;
    if (x3 < n3 && x1l < s) send[rp * blk + ((long long)x2l * n3 + x3) * s + x1l] = tile[threadIdx.x][i];
  }
}

// recv block r'' = [x2l][x3][x1l] (x1 = r'' s + x1l)  ->  T = [x2l < s2][x3 < n3][x1 < P1]
__global__ void unpack_AT_kernel(const double* __restrict__ recv, double* __restrict__ T, int s, int s2, int n3,
                                 int P1, long long blk) {
  const long long total = (long long)s2 * n3 * P1;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int x1 = (int)(e % P1);
    const long long row = e / P1;  // x2l * n3 + x3
    T[e] = recv[(long long)(x1 / s) * blk + row * s + (x1 % s)];
  }
}

// T = [x2l][x3][x1]  ->  send block r (x1 in [r s, (r+1) s)) = [x2l][x3][x1l]
__global__ void pack_TA_kernel(const double* __restrict__ T, double* __restrict__ send, int s, int s2, int n3,
                               int P1, int P, long long blk) {
  const long long total = (long long)P * blk;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / blk);
    const long long w = e % blk;
    const long long row = w / s;
    const int x1l = (int)(w % s);
    send[e] = T[row * P1 + (long long)r * s + x1l];
  }
}

// recv block r'' (x2 in [r'' s2, ...)) = [x2l][x3][x1l]  ->  A = [x1l][x2 < n2][x3 (+pad)]
// (planes x1l >= s_real are the x1 pad planes of the last slab: written as zeros -- with fused exchanges
// the send block position of the pad plane is not written by the x1 pass and holds stale data)
__global__ void unpack_TA_kernel(const double* __restrict__ recv, double* __restrict__ A, int s, int n2, int n3,
                                 int P3, int s2, long long blk, int s_real) {
  __shared__ double tile[32][33];
  const int x2 = blockIdx.z;
  const int x1_0 = blockIdx.x * 32, x3_0 = blockIdx.y * 32;
  const int rs = x2 / s2, x2l = x2 % s2;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int x3 = x3_0 + i, x1l = x1_0 + threadIdx.x;
    tile[i][threadIdx.x] = (x3 < n3 && x1l < s) ? recv[rs * blk + ((long long)x2l * n3 + x3) * s + x1l] : 0.0;
  }
  __syncthreads();
  if (x2 >= n2) return;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int x1l = x1_0 + i, x3 = x3_0 + threadIdx.x;
    if (x1l < s && x3 < n3) A[((long long)x1l * n2 + x2) * P3 + x3] = x1l < s_real ? tile[threadIdx.x][i] : 0.0;
  }
}

// sum of `count` doubles over up to 8 shard arrays, written back to every array (emulated allreduce)
struct Ptr8 {
  double* p[8];
};
__global__ void team_sum_kernel(Ptr8 a, int nl, int count) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    double s = 0.0;
    for (int l = 0; l < nl; ++l) s += a.p[l][i];
    for (int l = 0; l < nl; ++l) a.p[l][i] = s;
  }
}

}  // namespace

// ------------------------------------------------------------------------------ team
struct ShardBufs {
  Geom gA{}, gT{};
  int x1lo = 0, x2lo = 0, s_real = 0;
  double* W[4] = {nullptr, nullptr, nullptr, nullptr};
  double *Z = nullptr, *X = nullptr, *U0 = nullptr, *FP = nullptr, *FH = nullptr, *BUF = nullptr, *TMP = nullptr;
  double* T[4] = {nullptr, nullptr, nullptr, nullptr};  // layout T (unfused exchanges only)
  double* send[3] = {nullptr, nullptr, nullptr};        // all-to-all blocks [r][x2l][x3][x1l], P blk each
  double* recv[3] = {nullptr, nullptr, nullptr};
  std::vector<double*> V;
  double *vscale = nullptr, *h1 = nullptr, *h2 = nullptr, *part = nullptr, *nrm = nullptr, *red = nullptr;
  GmresState* st = nullptr;
};

struct rsfde_team {
  rsfde_ctx* tab = nullptr;  // tables of the global problem (no work vectors)
  int P = 1, rank0 = 0, nlocal = 1, s = 0, s2 = 0;
  // fused exchanges: the x1 passes read the receive blocks and write the send blocks directly
  // (segmented contiguous axis, PassParams::seg_lg), so only pack A->T and unpack T->A remain
  bool fused = false;
  long long blk = 0;
  // chunked exchanges (fused only): the slab's s planes are cut into nchunk sub-slabs of sc planes; the
  // all-to-all blocks are laid out [peer][chunk][x2l][x3][x1l < sc], so a (peer, chunk) piece is contiguous
  // and the x1 pass sees segments of sc planes.  Chunk c's exchange runs on the exchange stream xs while
  // the passes of chunk c+1 (way there) or the unpack and inverse DSTs of chunk c-1 (way back) run on
  // the caller's stream.
  int nchunk = 1, sc = 0;
  long long blkc = 0;
  cudaStream_t xs = nullptr;
  cudaEvent_t ev_s[8] = {}, ev_x[8] = {};
  std::vector<ShardBufs> sh;
  ncclComm_t comm = nullptr;
  void* h_flags = nullptr;
  std::string err;
  long long launches = 0, bytes = 0;
  std::vector<void*> allocs;
};

static rsfde_status tfail(rsfde_team* t, cudaError_t e, const char* what) {
  char b[256];
  snprintf(b, sizeof b, "%s: %s", what, cudaGetErrorString(e));
  if (t) t->err = b; else g_team_error = b;
  return e == cudaErrorMemoryAllocation ? RSFDE_E_NOMEM : RSFDE_E_CUDA;
}
static rsfde_status nfail(rsfde_team* t, ncclResult_t r, const char* what) {
  char b[256];
  snprintf(b, sizeof b, "%s: %s", what, g_nccl.ErrStr ? g_nccl.ErrStr(r) : "nccl error");
  if (t) t->err = b; else g_team_error = b;
  return RSFDE_E_NCCL;
}
#define TCK(expr, what)                                   \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return tfail(t, _e, what);     \
  } while (0)
#define TCKL(expr, what)                                  \
  do {                                                    \
    t->launches++;                                        \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return tfail(t, _e, what);     \
  } while (0)
#define TTRY(expr)                     \
  do {                                 \
    rsfde_status _s = (expr);          \
    if (_s != RSFDE_OK) return _s;     \
  } while (0)
#define TNC(expr, what)                                   \
  do {                                                    \
    ncclResult_t _r = (expr);                             \
    if (_r != ncclSuccess) return nfail(t, _r, what);     \
  } while (0)

static rsfde_status talloc(rsfde_team* t, double** p, size_t n) {
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(double));
  if (e != cudaSuccess) return tfail(t, e, "cudaMalloc");
  t->allocs.push_back(*p);
  t->bytes += (long long)(n * sizeof(double));
  e = cudaMemset(*p, 0, n * sizeof(double));
  if (e != cudaSuccess) return tfail(t, e, "cudaMemset");
  return RSFDE_OK;
}

// pass parameters of an axis of a local (sharded or transposed) geometry.  phys[i] = physical
// axis of local axis i; tables come from the global context in that permutation.
static PassParams local_params(const rsfde_team* t, const Geom& g, const int phys[3], int axis, const int coff[3]) {
  const rsfde_ctx* c = t->tab;
  PassParams p = rsfde_axis_params(c, phys[axis]);  // tables / coefficients of the pass axis
  p.geo = g;
  p.axis = axis;
  p.n = g.n[axis];
  p.N = p.n + 1;
  p.L = 2 * p.N;
  p.contiguous = axis == g.d - 1;
  long long stride = 1;
  if (!p.contiguous) {
    stride = g.P;
    for (int i = axis + 1; i < g.d - 1; ++i) stride *= g.n[i];
  }
  p.stride = stride;
  p.inner = stride;
  p.npairs = p.contiguous ? ((g.NP / g.P) + 1) / 2 : g.NP / p.n / 2;
  for (int i = 0; i < 3; ++i) {
    p.spec.eta[i] = c->eta[phys[i]];
    p.spec.q[i] = c->d_q[phys[i]];
    p.spec.lamH[i] = c->d_lamH[phys[i]];
    p.spec.tq[i] = c->d_tq[phys[i]];
    p.coff[i] = coff[i];
    p.cext[i] = c->n[phys[i]];
  }
  return p;
}

static const int kPhysA[3] = {0, 1, 2};  // layout A: x1, x2, x3
static const int kPhysT[3] = {1, 2, 0};  // layout T: x2, x3, x1

static PassParams paramsA(const rsfde_team* t, int l, int axis) {
  const int coff[3] = {t->sh[l].x1lo, 0, 0};
  return local_params(t, t->sh[l].gA, kPhysA, axis, coff);
}
static PassParams paramsT(const rsfde_team* t, int l) {
  const int coff[3] = {t->sh[l].x2lo, 0, 0};
  return local_params(t, t->sh[l].gT, kPhysT, 2, coff);
}

// sub-slab c (planes [c sc, (c+1) sc) of the local slab) of layout A: chunk geometry, global x1 offset
static PassParams paramsA_c(const rsfde_team* t, int l, int axis, int c) {
  if (t->nchunk == 1) return paramsA(t, l, axis);
  Geom g = t->sh[l].gA;
  g.n[0] = t->sc;
  g.NP = (long long)t->sc * g.n[1] * g.P;
  const int coff[3] = {t->sh[l].x1lo + c * t->sc, 0, 0};
  return local_params(t, g, kPhysA, axis, coff);
}
// element offset of sub-slab c inside a layout-A vector
static long long chunk_off(const rsfde_team* t, int l, int c) {
  const Geom& g = t->sh[l].gA;
  return (long long)c * t->sc * g.n[1] * g.P;
}

static ECoef ecoefA(const rsfde_team* t, int m) {
  ECoef e = rsfde_ecoef_at(t->tab, m);  // separable tables indexed by global coordinates
  return e;
}

// all-to-all of the shards' send buffers 0..nv-1 into their recv buffers (one NCCL group for all nv
// vectors: the two channels of the operator chain travel in one exchange)
// (chunk < 0: whole blocks; chunk c >= 0: the (peer, c) pieces of blkc elements)
static rsfde_status team_alltoall(rsfde_team* t, cudaStream_t s, int nv = 1, int chunk = -1) {
  const long long cnt = chunk < 0 ? t->blk : t->blkc;
  const long long coff = chunk < 0 ? 0 : (long long)chunk * t->blkc;
  const size_t bytes = (size_t)cnt * sizeof(double);
  if (!t->comm) {
    for (int v = 0; v < nv; ++v)
      for (int dst = 0; dst < t->P; ++dst)
        for (int src = 0; src < t->P; ++src)
          TCK(cudaMemcpyAsync(t->sh[dst].recv[v] + (long long)src * t->blk + coff,
                              t->sh[src].send[v] + (long long)dst * t->blk + coff, bytes, cudaMemcpyDeviceToDevice, s),
              "alltoall copy");
    return RSFDE_OK;
  }
  TNC(g_nccl.GroupStart(), "ncclGroupStart");
  for (int v = 0; v < nv; ++v)
    for (int peer = 0; peer < t->P; ++peer) {
      TNC(g_nccl.Send(t->sh[0].send[v] + (long long)peer * t->blk + coff, (size_t)cnt, ncclDouble, peer, t->comm, s),
          "ncclSend");
      TNC(g_nccl.Recv(t->sh[0].recv[v] + (long long)peer * t->blk + coff, (size_t)cnt, ncclDouble, peer, t->comm, s),
          "ncclRecv");
    }
  TNC(g_nccl.GroupEnd(), "ncclGroupEnd");
  return RSFDE_OK;
}

// in-place sum over ranks of count doubles at ptr(l) of every local shard
template <class F>
static rsfde_status team_allreduce(rsfde_team* t, F ptr, int count, cudaStream_t s) {
  if (!t->comm) {
    if (t->nlocal == 1) return RSFDE_OK;
    Ptr8 a{};
    for (int l = 0; l < t->nlocal; ++l) a.p[l] = ptr(l);
    TCKL((team_sum_kernel<<<1, 64, 0, s>>>(a, t->nlocal, count), cudaGetLastError()), "team sum");
    return RSFDE_OK;
  }
  TNC(g_nccl.AllReduce(ptr(0), ptr(0), (size_t)count, ncclDouble, ncclSum, t->comm, s), "ncclAllReduce");
  return RSFDE_OK;
}

static rsfde_status transpose_AT(rsfde_team* t, double* const* srcA, double* const* dstT, cudaStream_t s) {
  for (int l = 0; l < t->nlocal; ++l) {
    const ShardBufs& b = t->sh[l];
    const int n2 = t->tab->n[1], n3 = t->tab->n[2];
    dim3 grid((n3 + 31) / 32, (t->s + 31) / 32, t->P * t->s2);
    TCKL((pack_AT_kernel<<<grid, dim3(32, 8), 0, s>>>(srcA[l], b.send[0], t->s, n2, n3, b.gA.P, t->s2, t->blk),
          cudaGetLastError()),
         "pack A->T");
  }
  TTRY(team_alltoall(t, s));
  for (int l = 0; l < t->nlocal; ++l) {
    const ShardBufs& b = t->sh[l];
    TCKL((unpack_AT_kernel<<<stream_blocks(), 256, 0, s>>>(b.recv[0], dstT[l], t->s, t->s2, t->tab->n[2], b.gT.P, t->blk),
          cudaGetLastError()),
         "unpack A->T");
  }
  return RSFDE_OK;
}

static rsfde_status transpose_TA(rsfde_team* t, double* const* srcT, double* const* dstA, cudaStream_t s) {
  for (int l = 0; l < t->nlocal; ++l) {
    const ShardBufs& b = t->sh[l];
    TCKL((pack_TA_kernel<<<stream_blocks(), 256, 0, s>>>(srcT[l], b.send[0], t->s, t->s2, t->tab->n[2], b.gT.P, t->P, t->blk),
          cudaGetLastError()),
         "pack T->A");
  }
  TTRY(team_alltoall(t, s));
  for (int l = 0; l < t->nlocal; ++l) {
    const ShardBufs& b = t->sh[l];
    const int n2 = t->tab->n[1], n3 = t->tab->n[2];
    dim3 grid((t->s + 31) / 32, (n3 + 31) / 32, t->P * t->s2);
    TCKL((unpack_TA_kernel<<<grid, dim3(32, 8), 0, s>>>(b.recv[0], dstA[l], t->s, n2, n3, b.gA.P, t->s2, t->blk, b.s_real),
          cudaGetLastError()),
         "unpack T->A");
  }
  return RSFDE_OK;
}

// fused exchanges, way there: pack sub-slab c of layout-A vectors into the (peer, c) pieces of send
// buffers 0..nv-1 and start their exchange (one group) -- on the exchange stream when chunked, so that it
// runs under the passes of the next sub-slab
static rsfde_status pack_send_AT(rsfde_team* t, const std::vector<std::vector<const double*>>& srcA, int c,
                                 cudaStream_t s) {
  const int nv = (int)srcA.size();
  for (int v = 0; v < nv; ++v)
    for (int l = 0; l < t->nlocal; ++l) {
      const ShardBufs& b = t->sh[l];
      const int n2 = t->tab->n[1], n3 = t->tab->n[2];
      dim3 grid((n3 + 31) / 32, (t->sc + 31) / 32, t->P * t->s2);
      TCKL((pack_AT_kernel<<<grid, dim3(32, 8), 0, s>>>(srcA[v][l] + chunk_off(t, l, c), b.send[v] + (long long)c * t->blkc,
                                                         t->sc, n2, n3, b.gA.P, t->s2, t->blk),
            cudaGetLastError()),
           "pack A->T");
    }
  if (t->nchunk == 1) return team_alltoall(t, s, nv);
  TCK(cudaEventRecord(t->ev_s[c], s), "event");
  TCK(cudaStreamWaitEvent(t->xs, t->ev_s[c], 0), "wait");
  return team_alltoall(t, t->xs, nv, c);
}
// ... the caller's stream waits for every piece before the x1 pass
static rsfde_status join_exchange(rsfde_team* t, cudaStream_t s) {
  if (t->nchunk == 1) return RSFDE_OK;
  TCK(cudaEventRecord(t->ev_x[0], t->xs), "event");
  TCK(cudaStreamWaitEvent(s, t->ev_x[0], 0), "wait");
  return RSFDE_OK;
}
// way back, after the x1 pass wrote its send blocks: exchange piece by piece; as soon as piece c is
// here, unpack sub-slab c into layout A and (dst = true) run its inverse DSTs along x2 and x3
// (W0 -> W1 -> out) under the exchange of piece c+1
static rsfde_status exchange_unpack_TA(rsfde_team* t, double* const* dstA, bool dst, double* const* out,
                                       cudaStream_t s) {
  const int nc = t->nchunk;
  if (nc > 1) {
    TCK(cudaEventRecord(t->ev_s[0], s), "event");
    TCK(cudaStreamWaitEvent(t->xs, t->ev_s[0], 0), "wait");
    for (int c = 0; c < nc; ++c) {
      TTRY(team_alltoall(t, t->xs, 1, c));
      TCK(cudaEventRecord(t->ev_x[c], t->xs), "event");
    }
  } else {
    TTRY(team_alltoall(t, s, 1));
  }
  for (int c = 0; c < nc; ++c) {
    if (nc > 1) TCK(cudaStreamWaitEvent(s, t->ev_x[c], 0), "wait");
    for (int l = 0; l < t->nlocal; ++l) {
      const ShardBufs& b = t->sh[l];
      const int n2 = t->tab->n[1], n3 = t->tab->n[2];
      const int sreal = std::max(0, std::min(t->sc, b.s_real - c * t->sc));
      dim3 grid((t->sc + 31) / 32, (n3 + 31) / 32, t->P * t->s2);
      TCKL((unpack_TA_kernel<<<grid, dim3(32, 8), 0, s>>>(b.recv[0] + (long long)c * t->blkc, dstA[l] + chunk_off(t, l, c),
                                                           t->sc, n2, n3, b.gA.P, t->s2, t->blk, sreal),
            cudaGetLastError()),
           "unpack T->A");
    }
    if (!dst) continue;
    for (int l = 0; l < t->nlocal; ++l) {
      ShardBufs& b = t->sh[l];
      const long long off = chunk_off(t, l, c);
      PassParams p = paramsA_c(t, l, 1, c);
      p.X = b.W[0] + off;
      p.Y = b.W[1] + off;
      TCKL(launch_dst_pass(p, false, s), "dst x2");
      PassParams q = paramsA_c(t, l, 2, c);
      q.X = b.W[1] + off;
      q.Y = out[l] + off;
      TCKL(launch_dst_pass(q, false, s), "dst x3");
    }
  }
  return RSFDE_OK;
}
// x1-pass parameters on the receive blocks (segmented contiguous axis: segments of sc planes, one per
// (peer, chunk) piece)
static PassParams paramsT_seg(const rsfde_team* t, int l) {
  PassParams p = paramsT(t, l);
  int lg = 0;
  while ((1 << lg) < t->sc) ++lg;
  p.seg_lg = lg;
  p.seg_stride = t->blkc;
  return p;
}

struct TChain {
  int xmode = X_E_TIMES_R;
  std::vector<const double*> Xin, R, rscale, B;
  double etafac = 1.0, ycoef = 1.0, bcoef = 0.0;
  bool spectral = false;
  int spec = SPEC_PHAT;
  int m = 0;
};

// sharded operator chain (see the file header); out[l] in layout A, must not alias the inputs
static rsfde_status team_chain(rsfde_team* t, const TChain& a, double* const* out, cudaStream_t s) {
  const int nl = t->nlocal;
  const bool addB = !a.spectral && !a.B.empty() && a.B[0];
  // passes along x3 and x2 on sub-slab c (the whole slab when not chunked)
  auto passes_x3_x2 = [&](int c, bool chunked) -> rsfde_status {
    // pass along x3 (layout A, contiguous), first pass: X channel from the caller
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      const long long off = chunked ? chunk_off(t, l, c) : 0;
      PassParams p = chunked ? paramsA_c(t, l, 2, c) : paramsA(t, l, 2);
      p.xmode = a.xmode;
      p.X = a.xmode == X_INPUT ? a.Xin[l] + off : nullptr;
      p.R = a.R[l] + off;
      p.rscale = a.rscale.empty() ? nullptr : a.rscale[l];
      p.eta = a.etafac * t->tab->eta[2];
      if (a.xmode == X_E_TIMES_R) p.e = ecoefA(t, a.m);
      p.spec.kind = a.spec;
      p.Y = b.W[0] + off;
      p.C = b.W[1] + off;
      TCKL(launch_oper_pass(p, a.spectral, false, s), "pass x3");
    }
    // pass along x2 (layout A, strided)
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      const long long off = chunked ? chunk_off(t, l, c) : 0;
      PassParams p = chunked ? paramsA_c(t, l, 1, c) : paramsA(t, l, 1);
      p.xmode = X_INPUT;
      p.X = b.W[0] + off;
      p.R = b.W[1] + off;
      p.eta = a.etafac * t->tab->eta[1];
      p.spec.kind = a.spec;
      p.Y = b.W[2] + off;
      p.C = b.W[3] + off;
      TCKL(launch_oper_pass(p, a.spectral, false, s), "pass x2");
    }
    return RSFDE_OK;
  };
  if (t->fused) {
    // both channels (and B) in one exchange per sub-slab; the x1 pass reads the receive blocks and
    // writes the send blocks of the way back
    std::vector<std::vector<const double*>> src(addB ? 3 : 2, std::vector<const double*>(nl));
    for (int l = 0; l < nl; ++l) {
      src[0][l] = t->sh[l].W[2];
      src[1][l] = t->sh[l].W[3];
      if (addB) src[2][l] = a.B[l];
    }
    for (int c = 0; c < t->nchunk; ++c) {
      TTRY(passes_x3_x2(c, true));
      TTRY(pack_send_AT(t, src, c, s));
    }
    TTRY(join_exchange(t, s));
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      PassParams p = paramsT_seg(t, l);
      p.xmode = X_INPUT;
      p.X = b.recv[0];
      p.R = b.recv[1];
      p.eta = a.etafac * t->tab->eta[0];
      p.spec.kind = a.spec;
      p.ycoef = a.ycoef;
      p.B = addB ? b.recv[2] : nullptr;
      p.bcoef = a.bcoef;
      p.Y = b.send[0];
      TCKL(launch_oper_pass(p, a.spectral, true, s), "pass x1");
    }
    std::vector<double*> dstA(nl);
    for (int l = 0; l < nl; ++l) dstA[l] = a.spectral ? t->sh[l].W[0] : out[l];
    // (spectral: the inverse DSTs along x2 and x3 run per sub-slab inside)
    return exchange_unpack_TA(t, dstA.data(), a.spectral, out, s);
  }
  TTRY(passes_x3_x2(0, false));
  {
  // transpose both channels (and B) to layout T
  std::vector<double*> srcA(nl), dstT(nl);
  for (int l = 0; l < nl; ++l) { srcA[l] = t->sh[l].W[2]; dstT[l] = t->sh[l].T[0]; }
  TTRY(transpose_AT(t, srcA.data(), dstT.data(), s));
  for (int l = 0; l < nl; ++l) { srcA[l] = t->sh[l].W[3]; dstT[l] = t->sh[l].T[1]; }
  TTRY(transpose_AT(t, srcA.data(), dstT.data(), s));
  if (addB) {
    for (int l = 0; l < nl; ++l) { srcA[l] = const_cast<double*>(a.B[l]); dstT[l] = t->sh[l].T[2]; }
    TTRY(transpose_AT(t, srcA.data(), dstT.data(), s));
  }
  // last pass along x1 (layout T, contiguous)
  for (int l = 0; l < nl; ++l) {
    ShardBufs& b = t->sh[l];
    PassParams p = paramsT(t, l);
    p.xmode = X_INPUT;
    p.X = b.T[0];
    p.R = b.T[1];
    p.eta = a.etafac * t->tab->eta[0];
    p.spec.kind = a.spec;
    p.ycoef = a.ycoef;
    p.B = addB ? b.T[2] : nullptr;
    p.bcoef = a.bcoef;
    p.Y = b.T[3];
    TCKL(launch_oper_pass(p, a.spectral, true, s), "pass x1");
  }
  std::vector<double*> srcT(nl), dstA(nl);
  for (int l = 0; l < nl; ++l) {
    srcT[l] = t->sh[l].T[3];
    dstA[l] = a.spectral ? t->sh[l].W[0] : out[l];
  }
  TTRY(transpose_TA(t, srcT.data(), dstA.data(), s));
  }  // unfused
  if (!a.spectral) return RSFDE_OK;
  // inverse DSTs along x2 and x3 (layout A)
  for (int l = 0; l < nl; ++l) {
    ShardBufs& b = t->sh[l];
    PassParams p = paramsA(t, l, 1);
    p.X = b.W[0];
    p.Y = b.W[1];
    TCKL(launch_dst_pass(p, false, s), "dst x2");
    PassParams q = paramsA(t, l, 2);
    q.X = b.W[1];
    q.Y = out[l];
    TCKL(launch_dst_pass(q, false, s), "dst x3");
  }
  return RSFDE_OK;
}

// sharded S Lambda^{-1} S for the spectrum kind (in[l] -> out[l], layout A)
static rsfde_status team_precond(rsfde_team* t, int kind, double* const* in, double* const* out, cudaStream_t s) {
  const int nl = t->nlocal;
  // forward DSTs along x3 and x2 on sub-slab c (the whole slab when not chunked)
  auto dsts_x3_x2 = [&](int c, bool chunked) -> rsfde_status {
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      const long long off = chunked ? chunk_off(t, l, c) : 0;
      PassParams p = chunked ? paramsA_c(t, l, 2, c) : paramsA(t, l, 2);
      p.X = in[l] + off;
      p.Y = b.W[0] + off;
      TCKL(launch_dst_pass(p, false, s), "dst x3");
      PassParams q = chunked ? paramsA_c(t, l, 1, c) : paramsA(t, l, 1);
      q.X = b.W[0] + off;
      q.Y = b.W[1] + off;
      TCKL(launch_dst_pass(q, false, s), "dst x2");
    }
    return RSFDE_OK;
  };
  std::vector<double*> srcA(nl), dstT(nl), srcT(nl), dstA(nl);
  if (t->fused) {
    std::vector<std::vector<const double*>> src(1, std::vector<const double*>(nl));
    for (int l = 0; l < nl; ++l) src[0][l] = t->sh[l].W[1];
    for (int c = 0; c < t->nchunk; ++c) {
      TTRY(dsts_x3_x2(c, true));
      TTRY(pack_send_AT(t, src, c, s));
    }
    TTRY(join_exchange(t, s));
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      PassParams p = paramsT_seg(t, l);
      p.X = b.recv[0];
      p.Y = b.send[0];
      p.spec.kind = kind;
      TCKL(launch_dst_pass(p, true, s), "dst x1 (scaled)");
    }
    for (int l = 0; l < nl; ++l) dstA[l] = t->sh[l].W[0];
    return exchange_unpack_TA(t, dstA.data(), true, out, s);
  }
  TTRY(dsts_x3_x2(0, false));
  {
  for (int l = 0; l < nl; ++l) { srcA[l] = t->sh[l].W[1]; dstT[l] = t->sh[l].T[0]; }
  TTRY(transpose_AT(t, srcA.data(), dstT.data(), s));
  for (int l = 0; l < nl; ++l) {
    ShardBufs& b = t->sh[l];
    PassParams p = paramsT(t, l);
    p.X = b.T[0];
    p.Y = b.T[3];
    p.spec.kind = kind;
    TCKL(launch_dst_pass(p, true, s), "dst x1 (scaled)");
  }
  for (int l = 0; l < nl; ++l) { srcT[l] = t->sh[l].T[3]; dstA[l] = t->sh[l].W[0]; }
  TTRY(transpose_TA(t, srcT.data(), dstA.data(), s));
  }
  for (int l = 0; l < nl; ++l) {
    ShardBufs& b = t->sh[l];
    PassParams p = paramsA(t, l, 1);
    p.X = b.W[0];
    p.Y = b.W[1];
    TCKL(launch_dst_pass(p, false, s), "dst x2");
    PassParams q = paramsA(t, l, 2);
    q.X = b.W[1];
    q.Y = out[l];
    TCKL(launch_dst_pass(q, false, s), "dst x3");
  }
  return RSFDE_OK;
}

static rsfde_status team_ensure_basis(rsfde_team* t, int restart) {
  bool grew = false;
  for (auto& b : t->sh) {
    while ((int)b.V.size() < restart + 1) {
      double* v = nullptr;
      TTRY(talloc(t, &v, (size_t)b.gA.NP));
      b.V.push_back(v);
      grew = true;
    }
  }
  // talloc zeroes on the legacy default stream: finish that before the caller's stream reads the basis
  if (grew) TCK(cudaDeviceSynchronize(), "basis zeroing");
  return RSFDE_OK;
}

struct TFlags {
  int converged;
  int breakdown;
  double relres;
};

static rsfde_status team_flags(rsfde_team* t, TFlags* f, cudaStream_t s) {
  TCK(cudaMemcpyAsync(t->h_flags, t->sh[0].st, sizeof(TFlags), cudaMemcpyDeviceToHost, s), "flags");
  TCK(cudaStreamSynchronize(s), "sync");
  memcpy(f, t->h_flags, sizeof(TFlags));
  return RSFDE_OK;
}

// b = H E U0 - S_alpha U0 + tau FP into BUF (layout A)
static rsfde_status team_compute_b(rsfde_team* t, int m, cudaStream_t s) {
  TChain a;
  a.xmode = X_E_TIMES_R;
  for (auto& b : t->sh) { a.R.push_back(b.U0); a.B.push_back(b.FP); }
  a.etafac = -1.0;
  a.bcoef = t->tab->tau;
  a.m = m;
  std::vector<double*> out;
  for (auto& b : t->sh) out.push_back(b.BUF);
  return team_chain(t, a, out.data(), s);
}

static rsfde_status team_gmres(rsfde_team* t, int m, bool fast, bool have_b, const rsfde_gmres_cfg& cfg,
                               cudaStream_t s, int* iters_out, double* relres_out, int* conv_out) {
  const int restart = cfg.restart, nl = t->nlocal;
  const int max_iters = cfg.max_iters > 0 ? cfg.max_iters : 10 * restart;
  const int fixed = cfg.fixed_iters;
  const double tol = fixed > 0 ? -1.0 : cfg.tol;
  TTRY(team_ensure_basis(t, restart));
  const long long NP = t->sh[0].gA.NP;
  const int nb = reduction_blocks(NP, t->tab->nblk);
  int total = 0;
  bool first = true, converged = false;
  TFlags fl{0, 0, 1.0};
  std::vector<double*> outv(nl);
  while (true) {
    for (int l = 0; l < nl; ++l) outv[l] = t->sh[l].V[0];
    if (first && fast) {
      TChain a;
      a.xmode = X_INPUT;
      for (auto& b : t->sh) { a.Xin.push_back(b.FH); a.R.push_back(b.X); }
      a.etafac = -2.0;
      a.spectral = true;
      a.m = m;
      TTRY(team_chain(t, a, outv.data(), s));
    } else {
      if (!have_b) {
        TTRY(team_compute_b(t, m, s));
        have_b = true;
      }
      TChain a;
      a.xmode = X_E_TIMES_R;
      for (auto& b : t->sh) { a.R.push_back(b.X); a.B.push_back(b.BUF); }
      a.ycoef = -1.0;
      a.bcoef = 1.0;
      a.m = m;
      std::vector<double*> tmp(nl), tin(nl);
      for (int l = 0; l < nl; ++l) tmp[l] = t->sh[l].TMP;
      TTRY(team_chain(t, a, tmp.data(), s));
      TTRY(team_precond(t, SPEC_PHAT, tmp.data(), outv.data(), s));
    }
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      TCKL(launch_sumsq(b.V[0], b.nrm, NP, t->tab->nblk, s), "sumsq");
      TCKL(launch_reduce(b.nrm, nb, 1, b.red, s), "reduce");
    }
    TTRY(team_allreduce(t, [&](int l) { return t->sh[l].red; }, 1, s));
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      TCKL(launch_gmres_init(b.st, b.red, 1, b.vscale, first ? 1 : 0, s), "gmres init");
    }
    TTRY(team_flags(t, &fl, s));
    if (fl.converged) {
      converged = true;
      break;
    }
    int k = 0;
    for (int j = 0; j < restart; ++j) {
      const int J = j + 1;
      TChain a;
      a.xmode = X_E_TIMES_R;
      for (auto& b : t->sh) { a.R.push_back(b.V[j]); a.rscale.push_back(b.vscale + j); }
      a.spectral = true;
      a.m = m;
      std::vector<double*> zs(nl);
      for (int l = 0; l < nl; ++l) zs[l] = t->sh[l].Z;
      TTRY(team_chain(t, a, zs.data(), s));
      if (t->tab->ortho == ORTHO_DCGS2) {
        // DCGS2 (krylov_kernels.cu): local dots -> one allreduce of the 2j+2 sums -> re-orthogonalise /
        // Hessenberg on every rank; local update -> one allreduce of ||u'||^2 -> rotation, flags.
        // Two allreduces per Arnoldi step (CGS2: three).
        const int NT = 2 * j + 2;
        for (int l = 0; l < nl; ++l) {
          ShardBufs& b = t->sh[l];
          const double* const* Vp = (const double* const*)b.V.data();
          TCKL(launch_dcgs_dots(Vp, j, b.Z, b.part, NP, t->tab->nblk, nullptr, s), "dcgs dots");
          TCKL(launch_reduce(b.part, nb, NT, b.h1, s), "reduce dots");
        }
        TTRY(team_allreduce(t, [&](int l) { return t->sh[l].h1; }, NT, s));
        for (int l = 0; l < nl; ++l) {
          ShardBufs& b = t->sh[l];
          const double* const* Vp = (const double* const*)b.V.data();
          TCKL(launch_dcgs_finish_a(b.st, b.h1, 1, j, b.vscale, nullptr, s), "dcgs finish a");
          TCKL(launch_dcgs_update(Vp, j, b.st, b.Z, b.nrm, NP, t->tab->nblk, nullptr, s), "dcgs update");
          TCKL(launch_reduce(b.nrm, nb, 1, b.red, s), "reduce nrm");
        }
        TTRY(team_allreduce(t, [&](int l) { return t->sh[l].red; }, 1, s));
        for (int l = 0; l < nl; ++l) {
          ShardBufs& b = t->sh[l];
          TCKL(launch_dcgs_finish_b(b.st, b.red, 1, j, tol, b.vscale, nullptr, s), "dcgs finish b");
        }
        ++total;
        k = j + 1;
        TTRY(team_flags(t, &fl, s));
        const bool stop = fixed > 0 ? total >= fixed : fl.converged != 0;
        if (stop || fl.breakdown || total >= max_iters) break;
        continue;
      }
      for (int l = 0; l < nl; ++l) {
        ShardBufs& b = t->sh[l];
        const double* const* Vp = (const double* const*)b.V.data();
        TCKL(launch_dots(Vp, b.vscale, J, b.Z, b.part, NP, t->tab->nblk, s), "dots");
        TCKL(launch_reduce(b.part, nb, J, b.h1, s), "reduce h1");
      }
      TTRY(team_allreduce(t, [&](int l) { return t->sh[l].h1; }, J, s));
      for (int l = 0; l < nl; ++l) {
        ShardBufs& b = t->sh[l];
        const double* const* Vp = (const double* const*)b.V.data();
        TCKL(launch_dots_after_update(Vp, b.vscale, J, b.Z, b.h1, b.part, NP, t->tab->nblk, s), "dots2");
        TCKL(launch_reduce(b.part, nb, J, b.h2, s), "reduce h2");
      }
      TTRY(team_allreduce(t, [&](int l) { return t->sh[l].h2; }, J, s));
      for (int l = 0; l < nl; ++l) {
        ShardBufs& b = t->sh[l];
        const double* const* Vp = (const double* const*)b.V.data();
        TCKL(launch_update_norm(Vp, b.vscale, J, b.Z, b.h1, b.h2, b.V[j + 1], b.nrm, NP, t->tab->nblk, s), "update");
        TCKL(launch_reduce(b.nrm, nb, 1, b.red, s), "reduce nrm");
      }
      TTRY(team_allreduce(t, [&](int l) { return t->sh[l].red; }, 1, s));
      for (int l = 0; l < nl; ++l) {
        ShardBufs& b = t->sh[l];
        TCKL(launch_arnoldi_finish(b.st, b.h1, b.h2, b.red, 1, j, tol, b.vscale + j + 1, s), "finish");
      }
      ++total;
      k = j + 1;
      TTRY(team_flags(t, &fl, s));
      const bool stop = fixed > 0 ? total >= fixed : fl.converged != 0;
      if (stop || fl.breakdown || total >= max_iters) break;
    }
    for (int l = 0; l < nl; ++l) {
      ShardBufs& b = t->sh[l];
      TCKL(launch_gmres_solve_y(b.st, k, s), "solve y");
      const double* d_y = reinterpret_cast<const double*>(reinterpret_cast<const char*>(b.st) + offsetof(GmresState, y));
      const double* const* Vp = (const double* const*)b.V.data();
      TCKL(launch_axpy_basis(Vp, b.vscale, k, d_y, b.X, NP, s), "x update");
    }
    converged = fixed > 0 ? (total >= fixed || fl.breakdown != 0) : (fl.converged != 0 || fl.breakdown != 0);
    if (converged || total >= max_iters) break;
    first = false;
  }
  if (iters_out) *iters_out = total;
  if (relres_out) *relres_out = fl.relres;
  if (conv_out) *conv_out = converged ? 1 : 0;
  return RSFDE_OK;
}

// dense rows of the local ranks (virtual: the whole grid; one rank: its slab) <-> layout A
static rsfde_status team_load(rsfde_team* t, const double* src, double* const* dstA, cudaStream_t s) {
  const long long plane = (long long)t->tab->n[1] * t->tab->n[2];
  long long off = 0;
  for (int l = 0; l < t->nlocal; ++l) {
    ShardBufs& b = t->sh[l];
    Geom g = b.gA;
    g.n[0] = b.s_real;
    g.NP = (long long)b.s_real * g.n[1] * g.P;
    if (b.s_real > 0) TCKL(launch_pack(src + off, dstA[l], g, s), "pack");
    off += (long long)b.s_real * plane;
  }
  return RSFDE_OK;
}
static rsfde_status team_store(rsfde_team* t, double* const* srcA, double* dst, cudaStream_t s) {
  const long long plane = (long long)t->tab->n[1] * t->tab->n[2];
  long long off = 0;
  for (int l = 0; l < t->nlocal; ++l) {
    ShardBufs& b = t->sh[l];
    Geom g = b.gA;
    g.n[0] = b.s_real;
    g.NP = (long long)b.s_real * g.n[1] * g.P;
    if (b.s_real > 0) TCKL(launch_unpack(srcA[l], dst + off, g, s), "unpack");
    off += (long long)b.s_real * plane;
  }
  return RSFDE_OK;
}

// ------------------------------------------------------------------------------ ABI
extern "C" {

rsfde_status rsfde_nccl_unique_id(void* out128) {
  if (!out128) return RSFDE_E_CONFIG;
  if (!g_nccl.load()) {
    g_team_error = "libnccl.so.2 not found";
    return RSFDE_E_NCCL;
  }
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return RSFDE_E_NCCL;
  memcpy(out128, &id, sizeof id);
  return RSFDE_OK;
}

const char* rsfde_team_last_error(const rsfde_team* t) { return t ? t->err.c_str() : g_team_error.c_str(); }

void rsfde_team_destroy(rsfde_team* t) {
  if (!t) return;
  cudaDeviceSynchronize();
  for (void* p : t->allocs) cudaFree(p);
  if (t->h_flags) cudaFreeHost(t->h_flags);
  for (int c = 0; c < 8; ++c) {
    if (t->ev_s[c]) cudaEventDestroy(t->ev_s[c]);
    if (t->ev_x[c]) cudaEventDestroy(t->ev_x[c]);
  }
  if (t->xs) cudaStreamDestroy(t->xs);
  if (t->comm) g_nccl.CommDestroy(t->comm);
  if (t->tab) rsfde_destroy(t->tab);
  delete t;
}

rsfde_status rsfde_team_setup(rsfde_team** out, const rsfde_problem* p, int nranks, int rank, int nlocal,
                              const void* nccl_id, void* stream) {
  if (!out) return RSFDE_E_CONFIG;
  *out = nullptr;
  if (!p || p->d != 3) { g_team_error = "slab sharding needs d = 3"; return RSFDE_E_DIM; }
  if (p->e.kind != RSFDE_COEF_SEPARABLE) {
    // a dense e grid would need a per-rank slab layout (the pass kernels index it unsharded)
    g_team_error = "slab sharding supports the separable coefficient (RSFDE_COEF_SEPARABLE) only";
    return RSFDE_E_CONFIG;
  }
  if (nranks < 1 || nranks > 8 || (nlocal != 1 && nlocal != nranks) || rank < 0 || rank >= nranks ||
      (nlocal == nranks && rank != 0)) {
    g_team_error = "nranks in 1..8; nlocal = 1 (one rank per process) or nlocal = nranks (emulation, rank 0)";
    return RSFDE_E_CONFIG;
  }
  if ((p->n[0] + 1) % nranks || (p->n[1] + 1) % nranks) {
    g_team_error = "nranks must divide n1+1 and n2+1";
    return RSFDE_E_DIM;
  }
  if (nlocal < nranks && !nccl_id) { g_team_error = "multi-process sharding needs an NCCL unique id"; return RSFDE_E_CONFIG; }
  if (nccl_id && nlocal != 1) { g_team_error = "an NCCL communicator needs nlocal = 1"; return RSFDE_E_CONFIG; }
  rsfde_team* t = new rsfde_team();
  rsfde_status st = rsfde_setup_internal(&t->tab, p, stream, false);
  if (st != RSFDE_OK) {
    g_team_error = rsfde_last_error(nullptr);
    delete t;
    return st;
  }
  t->P = nranks;
  t->rank0 = rank;
  t->nlocal = nlocal;
  const int n1 = p->n[0], n2 = p->n[1], n3 = p->n[2];
  t->s = (n1 + 1) / nranks;
  t->s2 = (n2 + 1) / nranks;
  t->blk = (long long)t->s2 * n3 * t->s;
  // fused exchanges need segments of at most 256 planes (one TMA box per tile: nranks >= 2 at n1 = 511);
  // RSFDE_TEAM_UNFUSED=1 keeps the explicit layout-T transposes (test comparison)
  {
    const char* uf = getenv("RSFDE_TEAM_UNFUSED");
    t->fused = nranks >= 2 && t->s <= 256 && !(uf && *uf && strcmp(uf, "0"));
  }
  // chunked exchanges: RSFDE_TEAM_CHUNKS (default 4), reduced until sub-slabs of sc >= 2 planes divide s and
  // the x1 pass sees at most 256 segments (one TMA box dimension)
  t->nchunk = 1;
  if (t->fused) {
    int ch[2];
    long long piece = 0;
    if (rsfde_team_chunking(p->n, nranks, 0, ch, &piece) == RSFDE_OK) t->nchunk = ch[0];
  }
  t->sc = t->s / t->nchunk;
  t->blkc = t->blk / t->nchunk;
  t->sh.resize(nlocal);
  auto fail = [&](rsfde_status e) {
    g_team_error = t->err;
    rsfde_team_destroy(t);
    return e;
  };
  for (int l = 0; l < nlocal; ++l) {
    ShardBufs& b = t->sh[l];
    const int r = rank + l;
    int part[6];
    long long blk = 0;
    if ((st = rsfde_team_partition(p->n, nranks, r, part, &blk)) != RSFDE_OK || blk != t->blk) return fail(RSFDE_E_DIM);
    b.x1lo = part[0];
    b.x2lo = part[2];
    b.s_real = part[1];
    b.gA.d = 3;
    b.gA.n[0] = t->s;
    b.gA.n[1] = n2;
    b.gA.n[2] = n3;
    b.gA.P = n3 + 1;
    b.gA.NP = (long long)t->s * n2 * b.gA.P;
    b.gT.d = 3;
    b.gT.n[0] = t->s2;
    b.gT.n[1] = n3;
    b.gT.n[2] = n1;
    b.gT.P = n1 + 1;
    b.gT.NP = (long long)t->s2 * n3 * b.gT.P;
    double** va[] = {&b.W[0], &b.W[1], &b.W[2], &b.W[3], &b.Z, &b.X, &b.U0, &b.FP, &b.FH, &b.BUF, &b.TMP};
    for (double** v : va)
      if ((st = talloc(t, v, (size_t)b.gA.NP)) != RSFDE_OK) return fail(st);
    if (!t->fused)
      for (int i = 0; i < 4; ++i)
        if ((st = talloc(t, &b.T[i], (size_t)b.gT.NP)) != RSFDE_OK) return fail(st);
    for (int v = 0; v < (t->fused ? 3 : 1); ++v) {
      if ((st = talloc(t, &b.send[v], (size_t)(nranks * t->blk))) != RSFDE_OK) return fail(st);
      if ((st = talloc(t, &b.recv[v], (size_t)(nranks * t->blk))) != RSFDE_OK) return fail(st);
    }
    double** sm[] = {&b.vscale, &b.h1, &b.h2, &b.red};
    for (double** v : sm)
      if ((st = talloc(t, v, 128)) != RSFDE_OK) return fail(st);  // (DCGS2: 2j+2 <= 100 sums)
    if ((st = talloc(t, &b.part, (size_t)t->tab->nblk * 128)) != RSFDE_OK) return fail(st);
    if ((st = talloc(t, &b.nrm, (size_t)t->tab->nblk)) != RSFDE_OK) return fail(st);
    double* stp = nullptr;
    if ((st = talloc(t, &stp, (sizeof(GmresState) + 7) / 8)) != RSFDE_OK) return fail(st);
    b.st = reinterpret_cast<GmresState*>(stp);
  }
  if (cudaMallocHost(&t->h_flags, 64) != cudaSuccess) return fail(RSFDE_E_NOMEM);
  if (t->nchunk > 1) {
    if (cudaStreamCreateWithFlags(&t->xs, cudaStreamNonBlocking) != cudaSuccess) return fail(RSFDE_E_CUDA);
    for (int c = 0; c < 8; ++c)
      if (cudaEventCreateWithFlags(&t->ev_s[c], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&t->ev_x[c], cudaEventDisableTiming) != cudaSuccess)
        return fail(RSFDE_E_CUDA);
  }
  if (nccl_id) {
    if (!g_nccl.load()) {
      t->err = "libnccl.so.2 not found";
      return fail(RSFDE_E_NCCL);
    }
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof id);
    ncclResult_t r = g_nccl.CommInitRank(&t->comm, nranks, id, rank);
    if (r != ncclSuccess) return fail(nfail(t, r, "ncclCommInitRank"));
  }
  *out = t;
  return RSFDE_OK;
}

rsfde_status rsfde_team_chunking(const int n[3], int nranks, int requested, int out[2], long long* piece_elems) {
  if (!n || !out || nranks < 1 || nranks > 8) return RSFDE_E_CONFIG;
  if (n[0] < 1 || n[1] < 1 || n[2] < 1) return RSFDE_E_DIM;
  if ((n[0] + 1) % nranks || (n[1] + 1) % nranks) return RSFDE_E_DIM;
  const int s = (n[0] + 1) / nranks, s2 = (n[1] + 1) / nranks;
  int nc = requested;
  if (nc <= 0) {
    const char* ce = getenv("RSFDE_TEAM_CHUNKS");
    nc = ce ? atoi(ce) : 4;
  }
  if (nc < 1 || nranks == 1) nc = 1;
  if (nc > 8) nc = 8;
  while (nc > 1 && (s % nc || s / nc < 2 || (long long)nranks * nc > 256)) --nc;
  out[0] = nc;
  out[1] = s / nc;
  if (piece_elems) *piece_elems = (long long)s2 * n[2] * (s / nc);
  return RSFDE_OK;
}

rsfde_status rsfde_team_partition(const int n[3], int nranks, int rank, int out[6], long long* block_elems) {
  if (!n || !out || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks) return RSFDE_E_CONFIG;
  if (n[0] < 1 || n[1] < 1 || n[2] < 1) return RSFDE_E_DIM;
  if ((n[0] + 1) % nranks || (n[1] + 1) % nranks) return RSFDE_E_DIM;
  const int s = (n[0] + 1) / nranks, s2 = (n[1] + 1) / nranks;
  out[0] = rank * s;                                     // x1 slab (layout A)
  out[1] = std::max(0, std::min(s, n[0] - out[0]));      // (the last rank holds the x1 pad plane)
  out[2] = rank * s2;                                    // x2 slab (layout T)
  out[3] = std::max(0, std::min(s2, n[1] - out[2]));
  out[4] = s;
  out[5] = s2;
  if (block_elems) *block_elems = (long long)s2 * n[2] * s;  // all-to-all block [x2l < s2][x3 < n3][x1l < s]
  return RSFDE_OK;
}

rsfde_status rsfde_team_slab(const rsfde_team* t, int local, int* x1_lo, int* x1_count) {
  if (!t || local < 0 || local >= t->nlocal) return RSFDE_E_CONFIG;
  if (x1_lo) *x1_lo = t->sh[local].x1lo;
  if (x1_count) *x1_count = t->sh[local].s_real;
  return RSFDE_OK;
}

rsfde_status rsfde_team_matvec(rsfde_team* t, int op, int m, const double* x, double* y, void* stream) {
  if (!t) return RSFDE_E_CONFIG;
  if (!x || !y || x == y) return RSFDE_E_DIM;
  if (op != RSFDE_OP_K && op != RSFDE_OP_A) { t->err = "sharded matvec supports RSFDE_OP_K and RSFDE_OP_A"; return RSFDE_E_CONFIG; }
  if (m < 0 || m >= t->tab->M) return RSFDE_E_DOMAIN;
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::vector<double*> in(t->nlocal), outv(t->nlocal);
  for (int l = 0; l < t->nlocal; ++l) { in[l] = t->sh[l].BUF; outv[l] = t->sh[l].Z; }
  TTRY(team_load(t, x, in.data(), s));
  TChain a;
  a.xmode = X_E_TIMES_R;
  for (auto& b : t->sh) a.R.push_back(b.BUF);
  a.spectral = op == RSFDE_OP_K;
  a.m = m;
  TTRY(team_chain(t, a, outv.data(), s));
  return team_store(t, outv.data(), y, s);
}

rsfde_status rsfde_team_precond_apply(rsfde_team* t, int kind, const double* x, double* y, void* stream) {
  if (!t) return RSFDE_E_CONFIG;
  if (!x || !y || x == y) return RSFDE_E_DIM;
  int sk;
  switch (kind) {
    case RSFDE_PHAT_INV: sk = SPEC_PHAT; break;
    case RSFDE_PALPHA_INV: sk = SPEC_PALPHA; break;
    case RSFDE_PALPHA_INV_SQRT: sk = SPEC_PALPHA_SQRT; break;
    default: t->err = "unknown preconditioner"; return RSFDE_E_CONFIG;
  }
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  std::vector<double*> in(t->nlocal), outv(t->nlocal);
  for (int l = 0; l < t->nlocal; ++l) { in[l] = t->sh[l].BUF; outv[l] = t->sh[l].Z; }
  TTRY(team_load(t, x, in.data(), s));
  TTRY(team_precond(t, sk, in.data(), outv.data(), s));
  return team_store(t, outv.data(), y, s);
}

rsfde_status rsfde_team_solve_steps(rsfde_team* t, int m_begin, int m_count, double* u, const double* F, int F_static,
                                    const rsfde_gmres_cfg* cfg, rsfde_report* rep, void* stream) {
  if (!t) return RSFDE_E_CONFIG;
  if (!u) return RSFDE_E_DIM;
  if (m_begin < 0 || m_count < 0 || m_begin + m_count > t->tab->M) return RSFDE_E_DOMAIN;
  if (!cfg || cfg->restart < 1 || cfg->restart > 50 || cfg->form != RSFDE_FORM_A ||
      (cfg->fixed_iters <= 0 && !(cfg->tol >= 0.0))) {
    t->err = "bad GMRES configuration (sharded solver: A form, restart 1..50)";
    return RSFDE_E_CONFIG;
  }
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int nl = t->nlocal;
  long long Nloc = 0;
  for (auto& b : t->sh) Nloc += (long long)b.s_real * t->tab->n[1] * t->tab->n[2];
  cudaEvent_t e0, e1;
  TCK(cudaEventCreate(&e0), "event");
  TCK(cudaEventCreate(&e1), "event");
  TCK(cudaEventRecord(e0, s), "event");
  std::vector<double*> X(nl), FP(nl), FH(nl), U0(nl);
  for (int l = 0; l < nl; ++l) { X[l] = t->sh[l].X; FP[l] = t->sh[l].FP; FH[l] = t->sh[l].FH; U0[l] = t->sh[l].U0; }
  TTRY(team_load(t, u, X.data(), s));
  auto prepare_F = [&](const double* Fm) -> rsfde_status {
    for (int l = 0; l < nl; ++l) {
      if (!Fm) {
        TCK(cudaMemsetAsync(FP[l], 0, t->sh[l].gA.NP * sizeof(double), s), "memset");
      }
    }
    if (Fm) TTRY(team_load(t, Fm, FP.data(), s));
    TTRY(team_precond(t, SPEC_HINV, FP.data(), FH.data(), s));
    for (int l = 0; l < nl; ++l) TCKL(launch_axpby(0.0, FH[l], t->tab->tau, FH[l], t->sh[l].gA.NP, s), "scale");
    return RSFDE_OK;
  };
  if (!F || F_static) TTRY(prepare_F(F));
  long long total = 0;
  bool stopped = false;
  for (int k = 0; k < m_count; ++k) {
    const int m = m_begin + k;
    if (stopped) {
      if (rep && rep->iters) rep->iters[k] = -1;
      continue;
    }
    if (F && !F_static) TTRY(prepare_F(F + (long long)k * Nloc));
    for (int l = 0; l < nl; ++l)
      TCK(cudaMemcpyAsync(U0[l], X[l], t->sh[l].gA.NP * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy u0");
    int its = 0, conv = 0;
    double rr = 0;
    TTRY(team_gmres(t, m, true, false, *cfg, s, &its, &rr, &conv));
    total += its;
    if (rep) {
      if (rep->iters) rep->iters[k] = its;
      if (rep->final_relres) rep->final_relres[k] = rr;
      if (rep->converged) rep->converged[k] = (unsigned char)conv;
    }
    if (!conv) stopped = true;
  }
  TTRY(team_store(t, X.data(), u, s));
  TCK(cudaEventRecord(e1, s), "event");
  TCK(cudaEventSynchronize(e1), "event sync");
  float ms = 0;
  TCK(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->loop_seconds = ms * 1e-3;
    rep->setup_seconds = t->tab->setup_seconds;
    rep->total_iters = total;
  }
  return RSFDE_OK;
}

rsfde_status rsfde_team_compact_source(rsfde_team* t, int local, const double* f_closed_slab, double* F_slab,
                                       void* stream) {
  if (!t || local < 0 || local >= t->nlocal) return RSFDE_E_CONFIG;
  if (!f_closed_slab || !F_slab) return RSFDE_E_DIM;
  const ShardBufs& b = t->sh[local];
  if (b.s_real == 0) return RSFDE_OK;
  Geom g = b.gA;
  g.n[0] = b.s_real;
  g.NP = (long long)b.s_real * g.n[1] * g.P;
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  TCKL(launch_compact_source(f_closed_slab, F_slab, g, t->tab->alpha, s), "compact source");
  return RSFDE_OK;
}

long long rsfde_team_launch_count(const rsfde_team* t, int reset) {
  if (!t) return 0;
  const long long v = t->launches;
  if (reset) const_cast<rsfde_team*>(t)->launches = 0;
  return v;
}

}  // extern "C"
