// On-chip CN march for small 1-D problems (BASELINE C1: n = 255; SURVEY 8(d) "on-chip / latency: one
// CTA, whole run in shared memory").  One CTA of 1024 threads runs every CN step of Eq.(tls) and the
// whole tau-preconditioned GMRES solve of each step without returning to the host: the Krylov basis,
// the Hessenberg matrix and the 1-D tables live in shared memory, so an iteration costs a few
// microseconds instead of a host round trip per iteration.
//
// Operators (d = 1; the A form of DESIGN.md section 1):
//   A x      = H (e o x) + eta T x,   H = I + alpha/24 tridiag(1,-2,1),  T = [s_|i-j|] (FCD)
//   b        = H (e o u) - eta T u + tau F                                     (Eq.(tls))
//   P_hat^-1 = S Lambda^-1 S,  Lambda_k = ebar lambda^H_k + eta q_k
//   S_jk     = sqrt(2/(n+1)) sin(pi j k/(n+1))
// GMRES: left-preconditioned K = P_hat^-1 A from x0 = u^(m); first-cycle residual P_hat^-1(tau F - 2 eta
// T u) (b - A u, the H(e o u) terms cancel); CGS2; Givens; stop at |g_{j+1}| <= tol * beta_0.
// Dense products here (n^2 per operator) are cheaper than FFTs at these sizes and keep the CTA busy.
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.cuh"

namespace rsfde {

constexpr int kOnThreads = 1024;
constexpr int kOnWarps = kOnThreads / 32;

struct OnchipShared {
  // offsets (in doubles) into dynamic shared memory
  int V, x, u, w, t1, t2, e, sgen, lam, lh, sint, H, cs, sn, g, y, red, scr;
  int total;
};

__host__ __device__ inline OnchipShared onchip_layout(int n, int restart) {
  OnchipShared L;
  const int N2 = 2 * (n + 1);
  int o = 0;
  L.V = o; o += (restart + 1) * n;
  L.x = o; o += n;
  L.u = o; o += n;
  L.w = o; o += n;
  L.t1 = o; o += n;
  L.t2 = o; o += n;
  L.e = o; o += n;
  L.sgen = o; o += n;
  L.lam = o; o += n;
  L.lh = o; o += n;
  L.sint = o; o += N2;
  L.H = o; o += (restart + 1) * restart;
  L.cs = o; o += restart;
  L.sn = o; o += restart;
  L.g = o; o += restart + 1;
  L.y = o; o += restart;
  L.red = o; o += 2 * kOnWarps + 8;
  L.scr = o; o += 8 * n + 8;   // partial row sums of the split dense products
  L.total = o;
  return L;
}

size_t onchip_smem_bytes(int n, int restart) { return (size_t)onchip_layout(n, restart).total * sizeof(double); }

__device__ __forceinline__ double on_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum (all threads get the result)
__device__ __forceinline__ double on_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  v = on_warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wp] = v;
  __syncthreads();
  // every warp reduces the kOnWarps partials with shuffles (one load per lane instead of 32 per thread)
  return on_warp_sum(lane < kOnWarps ? red[lane] : 0.0);
}

struct OnchipCtx {
  const OnchipParams* P;
  double* sm;
  OnchipShared L;
  int n;
};

// out = T in   (T = [s_|i-j|], the FCD Toeplitz matrix).  T is persymmetric (J T J = T), so row n-1-i
// of T in is row i of T (J in): rows i and n-1-i share every coefficient load.  Up to 8 threads per row
// pair, each over an eighth of j (partial sums in scr).
__device__ __forceinline__ void on_toeplitz(const OnchipCtx& C, const double* in, double* out) {
  const double* s = C.sm + C.L.sgen;
  const int n = C.n, half = (n + 1) / 2;  // (n + 1 is a power of two: shifts and masks)
  double* scr = C.sm + C.L.scr;
  const int lh = __ffs(half) - 1;
  const int parts = min(8, max(1, (int)blockDim.x >> lh));
  const int chunk = (n + parts - 1) >> (__ffs(parts) - 1);
  for (int t = threadIdx.x; t < parts * half; t += blockDim.x) {
    const int i = t & (half - 1), pt = t >> lh;
    const int j0 = pt * chunk, j1 = min(n, j0 + chunk);
    double a1 = 0.0, a2 = 0.0;
    for (int j = j0; j < j1; ++j) {
      const double c = s[i > j ? i - j : j - i];
      a1 = fma(c, in[j], a1);
      a2 = fma(c, in[n - 1 - j], a2);
    }
    scr[pt * n + i] = a1;
    if (n - 1 - i != i) scr[pt * n + (n - 1 - i)] = a2;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = scr[i];
    for (int pt = 1; pt < parts; ++pt) acc += scr[pt * n + i];
    out[i] = acc;
  }
  __syncthreads();
}

// out = A in  (uses t1, t2)
__device__ void on_apply_A(const OnchipCtx& C, const double* in, double* out) {
  const int n = C.n;
  const OnchipParams& P = *C.P;
  double* t1 = C.sm + C.L.t1;
  double* t2 = C.sm + C.L.t2;
  const double* e = C.sm + C.L.e;
  for (int j = threadIdx.x; j < n; j += blockDim.x) t1[j] = e[j] * in[j];
  on_toeplitz(C, in, t2);  // (contains the barriers)
  const double h0 = 1.0 - P.alpha / 12.0, h1 = P.alpha / 24.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double hl = i > 0 ? t1[i - 1] : 0.0, hr = i + 1 < n ? t1[i + 1] : 0.0;
    out[i] = fma(h0, t1[i], fma(h1, hl + hr, P.eta * t2[i]));
  }
  __syncthreads();
}

// out = S in (orthonormal DST-I), k = 1..n stored at k-1; sint[i] = sin(pi i/(n+1)), i < 2(n+1).
// Outputs k and N-k (N = n+1) share their sines: sin(pi j (N-k)/N) = -(-1)^j sin(pi j k/N), so with
// A_k = sum over even j, B_k = sum over odd j of in_j sin(pi j k/N): out_k = A_k + B_k, out_{N-k} = B_k - A_k
// (half the sine recurrences of a row-by-row sum).  Up to 8 threads per k <= N/2, each over an eighth of
// j; sin(pi k j/N) advances by a rotation through pi k/N from an exact table value at the start of the
// chunk (a table gather per term would hit the same shared-memory bank for many k at once); <= n/8
// rotations keep the recurrence error below ~1e-15 relative.  N = n + 1 is a power of two (setup), so
// N is even and sint[i + N/2] = cos(pi i/N).
__device__ void on_dst(const OnchipCtx& C, const double* in, double* out) {
  const int n = C.n, N = n + 1, N2 = 2 * N, Q = N / 2;
  const double* st = C.sm + C.L.sint;
  double* scr = C.sm + C.L.scr;
  const double sc = sqrt(2.0 / (double)N);
  const int nk = N / 2;  // k = 1..N/2 computed directly, N-k from the same sums
  // (N, nk, N2 are powers of two: shifts and masks instead of divisions)
  const int lk = __ffs(nk) - 1, m2 = N2 - 1;
  const int parts = min(8, max(1, (int)blockDim.x >> lk));
  const int chunk = (n + parts - 1) >> (__ffs(parts) - 1);
  for (int t = threadIdx.x; t < parts * nk; t += blockDim.x) {
    const int k = (t & (nk - 1)) + 1, pt = t >> lk;
    const int j0 = 1 + pt * chunk, j1 = min(n, j0 + chunk - 1);
    const int i0 = (k * j0) & m2;
    double sv = st[i0], cv = st[(i0 + Q) & m2];
    const double sd = st[k], cd = st[(k + Q) & m2];
    double aE = 0.0, aO = 0.0;  // sums over even / odd j
    auto rot = [&]() {
      const double s2 = fma(sv, cd, cv * sd);
      cv = fma(cv, cd, -sv * sd);
      sv = s2;
    };
    int j = j0;
    if (j <= j1 && (j & 1)) {  // align to an even j
      aO = fma(sv, in[j - 1], aO);
      rot();
      ++j;
    }
    for (; j + 1 <= j1; j += 2) {
      aE = fma(sv, in[j - 1], aE);
      rot();
      aO = fma(sv, in[j], aO);
      rot();
    }
    if (j <= j1) aE = fma(sv, in[j - 1], aE);
    scr[pt * n + (k - 1)] = aE + aO;
    if (N - k != k) scr[pt * n + (N - k - 1)] = aO - aE;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    double acc = scr[k];
    for (int pt = 1; pt < parts; ++pt) acc += scr[pt * n + k];
    out[k] = sc * acc;
  }
  __syncthreads();
}

// out = P_hat^-1 in  (uses t2; in may alias out)
__device__ void on_apply_Pinv(const OnchipCtx& C, const double* in, double* out) {
  double* t2 = C.sm + C.L.t2;
  const double* lam = C.sm + C.L.lam;
  on_dst(C, in, t2);
  for (int k = threadIdx.x; k < C.n; k += blockDim.x) t2[k] /= lam[k];
  __syncthreads();
  on_dst(C, t2, out);
}

// the whole CN march of one system by one CTA (the single-system kernel and the batched kernel below)
__device__ __forceinline__ void onchip_march_body(const OnchipParams& P) {
  extern __shared__ double sm[];
  OnchipCtx C;
  C.P = &P;
  C.sm = sm;
  C.n = P.n;
  C.L = onchip_layout(P.n, P.restart);
  const OnchipShared& L = C.L;
  const int n = P.n, restart = P.restart, N2 = 2 * (n + 1);
  double* V = sm + L.V;
  double* x = sm + L.x;
  double* u = sm + L.u;
  double* w = sm + L.w;
  double* e = sm + L.e;
  double* H = sm + L.H;
  double* cs = sm + L.cs;
  double* sn = sm + L.sn;
  double* g = sm + L.g;
  double* y = sm + L.y;
  double* red = sm + L.red;
  __shared__ int s_flag;
  __shared__ double s_beta0, s_res;
  // ---- tables
  for (int i = threadIdx.x; i < N2; i += blockDim.x) sm[L.sint + i] = sinpi((double)i / (double)(n + 1));
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sm[L.sgen + i] = P.s[i];
    sm[L.lh + i] = P.lamH[i];
    sm[L.lam + i] = fma(P.ebar, P.lamH[i], P.eta * P.q[i]);  // Lambda_k = ebar lambda^H_k + eta q_k
    x[i] = P.X[i];
  }
  __syncthreads();
  const double h0 = 1.0 - P.alpha / 12.0, h1 = P.alpha / 24.0;
  for (int k = 0; k < P.m_count; ++k) {
    const int m = P.m_begin + k;
    const double* F = P.F ? P.F + (long long)k * P.F_stride : nullptr;
    // e(x, t_{m+1/2}) and u^(m)
    const double a = P.a_half[m], bb = P.b_half[m];
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      e[j] = a + bb * (P.g ? P.g[j] : 1.0) + (P.kk ? P.kk[j] : 0.0);
      u[j] = x[j];
    }
    __syncthreads();
    int total = 0;
    bool first = true, converged = false;
    double beta0 = 0.0, relres = 1.0;
    while (true) {
      // ---- residual r = P_hat^-1 (b - A x) into V_0
      double* r = V;
      if (first) {
        // b - A u = tau F - 2 eta T u   (x = u)
        double* t1 = sm + L.t1;
        on_toeplitz(C, u, t1);
        for (int i = threadIdx.x; i < n; i += blockDim.x) t1[i] = (F ? P.tau * F[i] : 0.0) - 2.0 * P.eta * t1[i];
        __syncthreads();
        on_apply_Pinv(C, t1, r);
      } else {
        // b = H(e o u) - eta T u + tau F ;  r = P^-1 (b - A x)
        on_apply_A(C, x, w);  // w = A x
        double* rb = V + n;   // basis slot 1 is free at residual time (restart >= 1)
        double* t1 = sm + L.t1;
        on_toeplitz(C, u, rb);  // rb = T u
        for (int j = threadIdx.x; j < n; j += blockDim.x) t1[j] = e[j] * u[j];
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const double hl = i > 0 ? t1[i - 1] : 0.0, hr = i + 1 < n ? t1[i + 1] : 0.0;
          const double b = fma(h0, t1[i], fma(h1, hl + hr, -P.eta * rb[i])) + (F ? P.tau * F[i] : 0.0);
          rb[i] = b - w[i];
        }
        __syncthreads();
        on_apply_Pinv(C, rb, r);
      }
      double part = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) part = fma(r[i], r[i], part);
      const double beta = sqrt(on_block_sum(part, red));
      if (first) beta0 = beta;
      if (beta == 0.0 || beta0 == 0.0) {
        converged = true;
        relres = 0.0;
        break;
      }
      const double ib = 1.0 / beta;
      for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] *= ib;
      if (threadIdx.x == 0) {
        g[0] = beta;
        for (int i = 1; i <= restart; ++i) g[i] = 0.0;
      }
      __syncthreads();
      int kk = 0;
      bool stop = false;
      for (int j = 0; j < restart; ++j) {
        double* vj = V + (long long)j * n;
        // w = K v_j
        on_apply_A(C, vj, w);
        on_apply_Pinv(C, w, w);
        // CGS2: two rounds of (h = V^T w, w -= V h); the dots one warp per basis vector
        for (int round = 0; round < 2; ++round) {
          for (int i = threadIdx.x >> 5; i <= j; i += kOnWarps) {
            const double* vi = V + (long long)i * n;
            double acc = 0.0;
            for (int t = threadIdx.x & 31; t < n; t += 32) acc = fma(vi[t], w[t], acc);
            acc = on_warp_sum(acc);
            if ((threadIdx.x & 31) == 0) {
              if (round == 0) H[j * (restart + 1) + i] = acc;
              else H[j * (restart + 1) + i] += acc;
              y[i] = acc;  // this round's coefficients
            }
          }
          __syncthreads();
          for (int t = threadIdx.x; t < n; t += blockDim.x) {
            double acc = w[t];
            for (int i = 0; i <= j; ++i) acc = fma(-y[i], V[(long long)i * n + t], acc);
            w[t] = acc;
          }
          __syncthreads();
        }
        part = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) part = fma(w[i], w[i], part);
        const double hnext = sqrt(on_block_sum(part, red));
        // Givens on column j (thread 0)
        if (threadIdx.x == 0) {
          double* hc = H + j * (restart + 1);
          hc[j + 1] = hnext;
          for (int i = 0; i < j; ++i) {
            const double t = cs[i] * hc[i] + sn[i] * hc[i + 1];
            hc[i + 1] = -sn[i] * hc[i] + cs[i] * hc[i + 1];
            hc[i] = t;
          }
          const double den = hypot(hc[j], hc[j + 1]);
          cs[j] = hc[j] / den;
          sn[j] = hc[j + 1] / den;
          hc[j] = den;
          hc[j + 1] = 0.0;
          g[j + 1] = -sn[j] * g[j];
          g[j] = cs[j] * g[j];
          const int tot = total + 1;
          const bool conv = fabs(g[j + 1]) <= P.tol * beta0;
          s_res = fabs(g[j + 1]) / beta0;
          s_flag = (conv ? 1 : 0) | (hnext == 0.0 ? 2 : 0) | (tot >= P.max_iters ? 4 : 0);
        }
        __syncthreads();
        ++total;
        kk = j + 1;
        const int fl = s_flag;
        relres = s_res;
        if (fl) {
          stop = (fl & 1) != 0 || (fl & 2) != 0;
          break;
        }
        const double ih = 1.0 / hnext;
        double* vn = V + (long long)(j + 1) * n;
        for (int t = threadIdx.x; t < n; t += blockDim.x) vn[t] = w[t] * ih;
        __syncthreads();
      }
      // y = R^-1 g (thread 0), x += V y
      if (threadIdx.x == 0) {
        for (int i = kk - 1; i >= 0; --i) {
          double acc = g[i];
          for (int l = i + 1; l < kk; ++l) acc -= H[l * (restart + 1) + i] * y[l];
          y[i] = acc / H[i * (restart + 1) + i];
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < n; t += blockDim.x) {
        double acc = x[t];
        for (int i = 0; i < kk; ++i) acc = fma(y[i], V[(long long)i * n + t], acc);
        x[t] = acc;
      }
      __syncthreads();
      if (stop) {
        converged = true;
        break;
      }
      if (total >= P.max_iters) break;
      first = false;
    }
    if (threadIdx.x == 0) {
      P.iters[k] = total;
      P.relres[k] = relres;
      P.conv[k] = converged ? 1 : 0;
    }
    if (!converged) {
      // the march stops at a step that did not converge (as rsfde_solve_steps)
      for (int kk2 = k + 1 + (int)threadIdx.x; kk2 < P.m_count; kk2 += blockDim.x) {
        P.iters[kk2] = -1;
        P.conv[kk2] = 0;
        P.relres[kk2] = 0.0;
      }
      break;
    }
    (void)beta0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) P.X[i] = x[i];
}

__global__ void __launch_bounds__(kOnThreads, 1) onchip_1d_kernel(const OnchipParams P) { onchip_march_body(P); }

// many independent 1-D systems per launch (the alpha / N sweeps of Tables 1-3,
// P:528-636), one CTA per system, each with its own parameters, tables, source and solution
__global__ void __launch_bounds__(kOnThreads, 1) onchip_1d_batch_kernel(const OnchipParams* __restrict__ Ps) {
  __shared__ OnchipParams sP;
  if (threadIdx.x == 0) sP = Ps[blockIdx.x];
  __syncthreads();
  onchip_march_body(sP);
}

cudaError_t launch_onchip_1d_batch(const OnchipParams* d_params, int count, size_t smem, cudaStream_t s) {
  struct Tag {};
  const int attr = per_device_once<Tag>([](int) -> int {
    return (int)cudaFuncSetAttribute(onchip_1d_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  });
  if (attr != (int)cudaSuccess) return attr < 0 ? cudaErrorInvalidDevice : (cudaError_t)attr;
  if (smem > 220 * 1024 || count < 1) return cudaErrorInvalidValue;
  onchip_1d_batch_kernel<<<count, kOnThreads, smem, s>>>(d_params);
  return cudaGetLastError();
}

cudaError_t launch_onchip_1d(const OnchipParams& p, cudaStream_t s) {
  const size_t smem = onchip_smem_bytes(p.n, p.restart);
  struct Tag {};
  const int attr = per_device_once<Tag>([](int) -> int {
    return (int)cudaFuncSetAttribute(onchip_1d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  });
  if (attr != (int)cudaSuccess) return attr < 0 ? cudaErrorInvalidDevice : (cudaError_t)attr;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  onchip_1d_kernel<<<1, kOnThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rsfde
