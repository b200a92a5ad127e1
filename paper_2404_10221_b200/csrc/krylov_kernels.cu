// GMRES / Arnoldi machinery (FP64, sm_100a): classical Gram-Schmidt with one
// re-orthogonalisation (CGS2) as streaming multi-dot / multi-axpy kernels with
// deterministic two-level reductions, the Hessenberg least-squares update by Givens
// rotations on the device, and small layout/utility kernels.
//
// GMRES is [Saad86]; the stopping rule |g_{j+1}| <= tol*beta_0 is P:513.
// Basis vectors are stored unnormalised with a per-vector scale s_i (v_i = s_i V_i), so
// normalisation never costs a pass; every kernel multiplies by s_i on the fly.
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.cuh"

namespace rsfde {

constexpr int kMaxBasis = 52;
struct BasisPtrs {
  const double* V[kMaxBasis];
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-reduce JP accumulators (only i < J used) and write partial[blockIdx.x*J + i]*scale_i
template <int JP>
__device__ __forceinline__ void block_reduce_store(double (&acc)[JP], int J, double* partial,
                                                   const double* scale) {
  __shared__ double red[8][kMaxBasis];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < JP; ++i) {
    if (i < J) {
      const double s = warp_sum(acc[i]);
      if (lane == 0) red[w][i] = s;
    }
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < J; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s += red[k][i];
    partial[(long long)blockIdx.x * J + i] = scale ? s * scale[i] : s;
  }
}

template <int JP>
__global__ void __launch_bounds__(256) dots_kernel(BasisPtrs b, const double* __restrict__ vscale, int J,
                                                   const double* __restrict__ z, double* __restrict__ partial,
                                                   long long n2) {
  double acc[JP];
#pragma unroll
  for (int i = 0; i < JP; ++i) acc[i] = 0.0;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (long long)gridDim.x * blockDim.x) {
    const double2 zz = __ldg(z2 + e);
    double2 vv[JP];  // all loads first (more bytes in flight per thread), then the FMAs
#pragma unroll
    for (int i = 0; i < JP; ++i)
      if (i < J) vv[i] = __ldg(reinterpret_cast<const double2*>(b.V[i]) + e);
#pragma unroll
    for (int i = 0; i < JP; ++i)
      if (i < J) acc[i] = fma(vv[i].x, zz.x, fma(vv[i].y, zz.y, acc[i]));
  }
  block_reduce_store<JP>(acc, J, partial, vscale);
}

// round-2 dots of CGS2 without materialising z' = z - sum c_l s_l V_l
template <int JP>
__global__ void __launch_bounds__(256) dots_after_update_kernel(BasisPtrs b, const double* __restrict__ vscale, int J,
                                                                const double* __restrict__ z,
                                                                const double* __restrict__ coef,
                                                                double* __restrict__ partial, long long n2) {
  __shared__ double cs[kMaxBasis];
  for (int i = threadIdx.x; i < J; i += blockDim.x) cs[i] = coef[i] * vscale[i];
  __syncthreads();
  double acc[JP], ncs[JP];
#pragma unroll
  for (int i = 0; i < JP; ++i) {
    acc[i] = 0.0;
    ncs[i] = i < J ? -cs[i] : 0.0;  // coefficients in registers (not re-read from shared memory per element)
  }
  // two elements per thread (16-byte loads: the scalar version reached 3.6 TB/s, the others 5.5-6)
  const double2* z2 = reinterpret_cast<const double2*>(z);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (long long)gridDim.x * blockDim.x) {
    double2 vv[JP];
    double2 zz = __ldg(z2 + e);
#pragma unroll
    for (int i = 0; i < JP; ++i)
      if (i < J) vv[i] = __ldg(reinterpret_cast<const double2*>(b.V[i]) + e);
#pragma unroll
    for (int i = 0; i < JP; ++i) {
      if (i < J) {
        zz.x = fma(ncs[i], vv[i].x, zz.x);
        zz.y = fma(ncs[i], vv[i].y, zz.y);
      }
    }
#pragma unroll
    for (int i = 0; i < JP; ++i)
      if (i < J) acc[i] = fma(vv[i].x, zz.x, fma(vv[i].y, zz.y, acc[i]));
  }
  block_reduce_store<JP>(acc, J, partial, vscale);
}

// out = z - sum_l (c1_l + c2_l) s_l V_l ; partial[b] = sum out^2
template <int JP>
__global__ void __launch_bounds__(256) update_norm_kernel(BasisPtrs b, const double* __restrict__ vscale, int J,
                                                          const double* __restrict__ z, const double* __restrict__ c1,
                                                          const double* __restrict__ c2, double* __restrict__ out,
                                                          double* __restrict__ partial, long long n2) {
  __shared__ double cs[kMaxBasis];
  for (int i = threadIdx.x; i < J; i += blockDim.x) cs[i] = (c1[i] + (c2 ? c2[i] : 0.0)) * vscale[i];
  __syncthreads();
  double acc[1] = {0.0};
  double ncs[JP];
#pragma unroll
  for (int i = 0; i < JP; ++i) ncs[i] = i < J ? -cs[i] : 0.0;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  double2* o2 = reinterpret_cast<double2*>(out);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (long long)gridDim.x * blockDim.x) {
    double2 zz = __ldg(z2 + e);
    double2 vv[JP];
#pragma unroll
    for (int i = 0; i < JP; ++i)
      if (i < J) vv[i] = __ldg(reinterpret_cast<const double2*>(b.V[i]) + e);
#pragma unroll
    for (int i = 0; i < JP; ++i) {
      if (i < J) {
        zz.x = fma(ncs[i], vv[i].x, zz.x);
        zz.y = fma(ncs[i], vv[i].y, zz.y);
      }
    }
    o2[e] = zz;
    acc[0] = fma(zz.x, zz.x, fma(zz.y, zz.y, acc[0]));
  }
  block_reduce_store<1>(acc, 1, partial, nullptr);
}

template <int JP>
__global__ void __launch_bounds__(256) axpy_basis_kernel(BasisPtrs b, const double* __restrict__ vscale, int J,
                                                         const double* __restrict__ y, double* __restrict__ x,
                                                         long long n2) {
  __shared__ double cs[kMaxBasis];
  for (int i = threadIdx.x; i < J; i += blockDim.x) cs[i] = y[i] * vscale[i];
  __syncthreads();
  double csr[JP];
#pragma unroll
  for (int i = 0; i < JP; ++i) csr[i] = i < J ? cs[i] : 0.0;
  double2* x2 = reinterpret_cast<double2*>(x);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (long long)gridDim.x * blockDim.x) {
    double2 xx = x2[e];
    double2 vv[JP];
#pragma unroll
    for (int i = 0; i < JP; ++i)
      if (i < J) vv[i] = __ldg(reinterpret_cast<const double2*>(b.V[i]) + e);
#pragma unroll
    for (int i = 0; i < JP; ++i) {
      if (i < J) {
        xx.x = fma(csr[i], vv[i].x, xx.x);
        xx.y = fma(csr[i], vv[i].y, xx.y);
      }
    }
    x2[e] = xx;
  }
}

__global__ void __launch_bounds__(256) sumsq_kernel(const double* __restrict__ z, double* __restrict__ partial, long long n2) {
  double acc[1] = {0.0};
  const double2* z2 = reinterpret_cast<const double2*>(z);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (long long)gridDim.x * blockDim.x) {
    const double2 zz = __ldg(z2 + e);
    acc[0] = fma(zz.x, zz.x, fma(zz.y, zz.y, acc[0]));
  }
  block_reduce_store<1>(acc, 1, partial, nullptr);
}

__global__ void __launch_bounds__(256) axpby_kernel(double a, const double* __restrict__ x, double bb, double* __restrict__ y,
                                                    long long n2) {
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double2* y2 = reinterpret_cast<double2*>(y);
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (long long)gridDim.x * blockDim.x) {
    const double2 xx = __ldg(x2 + e);
    double2 yy = y2[e];
    yy.x = fma(a, xx.x, bb * yy.x);
    yy.y = fma(a, xx.y, bb * yy.y);
    y2[e] = yy;
  }
}

// out[i] = sum_b partial[b*J + i], fixed order: warp w handles i = w, w+8, ...
__global__ void __launch_bounds__(256) reduce_kernel(const double* __restrict__ partial, int nblk, int J, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = w; i < J; i += 8) {
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[(long long)b * J + i];
    s = warp_sum(s);
    if (lane == 0) out[i] = s;
  }
}

__device__ double block_sum_partials(const double* partial, int nblk) {
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) s += partial[b];
  s = warp_sum(s);
  if (lane == 0) red[w] = s;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
  __syncthreads();
  return t;
}

constexpr int kLdH = 52;

__global__ void __launch_bounds__(256) arnoldi_finish_kernel(GmresState* st, const double* __restrict__ h1,
                                                             const double* __restrict__ h2, const double* __restrict__ pnrm,
                                                             int nblk, int j, double tol, double* vscale_next) {
  const int J = j + 1;
  const double nrm2 = block_sum_partials(pnrm, nblk);
  if (threadIdx.x != 0) return;
  double* H = st->H;
  for (int i = 0; i < J; ++i) {
    st->hsum[i] = h1[i] + h2[i];
    H[i + j * kLdH] = st->hsum[i];
  }
  const double beta = sqrt(nrm2);
  H[(j + 1) + j * kLdH] = beta;
  for (int i = 0; i < j; ++i) {
    const double a = H[i + j * kLdH], b = H[(i + 1) + j * kLdH];
    H[i + j * kLdH] = st->cs[i] * a + st->sn[i] * b;
    H[(i + 1) + j * kLdH] = -st->sn[i] * a + st->cs[i] * b;
  }
  const double a = H[j + j * kLdH], b = H[(j + 1) + j * kLdH];
  const double den = hypot(a, b);
  st->cs[j] = a / den;
  st->sn[j] = b / den;
  H[j + j * kLdH] = den;
  H[(j + 1) + j * kLdH] = 0.0;
  st->g[j + 1] = -st->sn[j] * st->g[j];
  st->g[j] = st->cs[j] * st->g[j];
  st->relres = fabs(st->g[j + 1]) / st->beta0;
  st->converged = st->relres <= tol ? 1 : 0;
  st->breakdown = (beta == 0.0) ? 1 : 0;
  *vscale_next = beta > 0.0 ? 1.0 / beta : 0.0;
}

__global__ void gmres_init_kernel(GmresState* st, const double* __restrict__ pnrm, int nblk, double* vscale0,
                                  int first_cycle, GraphCond gc) {
  const double nrm2 = block_sum_partials(pnrm, nblk);
  if (threadIdx.x != 0) return;
  if (gc.on) {  // graph-captured cycle: Arnoldi steps run while r0 != 0; no column yet
    st->steps = 0;
    cudaGraphSetConditional(gc.h_cont, nrm2 > 0.0 ? 1u : 0u);
  }
  const double beta = sqrt(nrm2);
  for (int i = 0; i < kLdH; ++i) st->g[i] = 0.0;
  st->g[0] = beta;
  if (first_cycle) st->beta0 = beta;
  st->relres = st->beta0 > 0.0 ? beta / st->beta0 : 0.0;
  st->converged = (beta == 0.0) ? 1 : 0;
  st->breakdown = 0;
  st->kcols = -1;
  st->nu = 1.0;
  *vscale0 = beta > 0.0 ? 1.0 / beta : 0.0;
}

__global__ void gmres_solve_y_kernel(GmresState* st, int k) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double* H = st->H;
  // DCGS2 records the usable column count on the device (kcols < 0: the host's k)
  if (st->kcols >= 0 && st->kcols < k) {
    for (int i = st->kcols; i < k; ++i) st->y[i] = 0.0;
    k = st->kcols;
  }
  for (int i = k - 1; i >= 0; --i) {
    double s = st->g[i];
    for (int l = i + 1; l < k; ++l) s -= H[i + l * kLdH] * st->y[l];
    st->y[i] = s / H[i + i * kLdH];
  }
}

// ------------------------------------------------------------------------------ DCGS2 Arnoldi
// Classical Gram-Schmidt with delayed re-orthogonalisation ("DCGS2": the second CGS pass of vector j
// runs in iteration j+1, fused with the first pass of the next vector, the norm by Pythagoras), so an
// Arnoldi step streams the basis twice instead of three times: one dots pass (j+2 vectors read) and
// one update pass (j+2 read, 2 written) against CGS2's 3j+7 vectors.  In exact arithmetic the
// iterates are those of CGS2 / MGS GMRES [Saad86]; the convergence test uses the
// once-orthogonalised norm of the newest vector (it differs from the twice-orthogonalised one at
// rounding level).

// chunk of up to CH basis vectors [i0, i0+cnt): a_l = V_{i0+l}.u, c_l = V_{i0+l}.w; with `first` also
// sigma = u.u and gamma = u.w.  u = V_j, all values unscaled (finish_a applies the lazy scales).
template <int CH>
__global__ void __launch_bounds__(256, 2) dcgs_dots_kernel(BasisPtrs b, int i0, int cnt, int j, int first,
                                                        const double* __restrict__ w, double* __restrict__ partial,
                                                        int NT, long long n2, const int* skip) {
  if (skip_launch(skip)) return;
  double acc_a[CH], acc_c[CH];
  double sig = 0.0, gam = 0.0;
#pragma unroll
  for (int l = 0; l < CH; ++l) acc_a[l] = acc_c[l] = 0.0;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const double2* u2 = reinterpret_cast<const double2*>(b.V[j]);
  // two grid-stride elements per iteration: all loads of both first (twice the bytes in flight)
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < n2; e0 += 2 * stride) {
    const bool two = e0 + stride < n2;
    double2 ww[2], uu[2], vv[2][CH];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long e = e0 + h * stride;
      const bool ok = h == 0 || two;
      ww[h] = ok ? __ldg(w2 + e) : make_double2(0.0, 0.0);
      uu[h] = ok ? __ldg(u2 + e) : make_double2(0.0, 0.0);
#pragma unroll
      for (int l = 0; l < CH; ++l)
        if (l < cnt) vv[h][l] = ok ? __ldg(reinterpret_cast<const double2*>(b.V[i0 + l]) + e) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int l = 0; l < CH; ++l) {
        if (l < cnt) {
          acc_a[l] = fma(vv[h][l].x, uu[h].x, fma(vv[h][l].y, uu[h].y, acc_a[l]));
          acc_c[l] = fma(vv[h][l].x, ww[h].x, fma(vv[h][l].y, ww[h].y, acc_c[l]));
        }
      }
      if (first) {
        sig = fma(uu[h].x, uu[h].x, fma(uu[h].y, uu[h].y, sig));
        gam = fma(uu[h].x, ww[h].x, fma(uu[h].y, ww[h].y, gam));
      }
    }
  }
  // block reduction of 2 cnt (+2) values, fixed order
  __shared__ double red[8][2 * CH + 2];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int l = 0; l < CH; ++l) {
    if (l < cnt) {
      const double sa = warp_sum(acc_a[l]), sc = warp_sum(acc_c[l]);
      if (lane == 0) { red[wp][l] = sa; red[wp][CH + l] = sc; }
    }
  }
  if (first) {
    const double ss = warp_sum(sig), sg = warp_sum(gam);
    if (lane == 0) { red[wp][2 * CH] = ss; red[wp][2 * CH + 1] = sg; }
  }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double* out = partial + (long long)blockIdx.x * NT;
  for (int t = threadIdx.x; t < 2 * CH + 2; t += blockDim.x) {
    int dst;
    if (t < CH) dst = t < cnt ? i0 + t : -1;
    else if (t < 2 * CH) dst = (t - CH) < cnt ? j + i0 + (t - CH) : -1;
    else dst = first ? 2 * j + (t - 2 * CH) : -1;
    if (dst < 0) continue;
    double v = 0.0;
    for (int k = 0; k < nw; ++k) v += red[k][t];
    out[dst] = v;
  }
}

// chunk [i0, i0+cnt) of the update: q_j += sum cq_i V_i (j > 0), u' += sum cu_i V_i.  The first chunk
// starts from q_j = cq_j V_j and u' = w + cu_j V_j, later chunks from the partial outputs; the last
// chunk also writes the partial sums of ||u'||^2.
template <int CH>
__global__ void __launch_bounds__(256, 2) dcgs_update_kernel(BasisPtrs b, int i0, int cnt, int j, int first, int last,
                                                          const GmresState* __restrict__ st,
                                                          const double* __restrict__ w, double* outq, double* outu,
                                                          double* __restrict__ partial, long long n2, const int* skip) {
  if (skip_launch(skip)) return;
  double cq[CH], cu[CH];
#pragma unroll
  for (int l = 0; l < CH; ++l) {
    cq[l] = l < cnt ? st->cq[i0 + l] : 0.0;
    cu[l] = l < cnt ? st->cu[i0 + l] : 0.0;
  }
  const double cqj = st->cq[j], cuj = st->cu[j];
  const bool wq = j > 0;
  double acc[1] = {0.0};
  const double2* w2 = reinterpret_cast<const double2*>(w);
  double2* q2 = reinterpret_cast<double2*>(outq);
  double2* u2 = reinterpret_cast<double2*>(outu);
  // two grid-stride elements per iteration: all loads of both first (twice the bytes in flight)
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < n2; e0 += 2 * stride) {
    const bool two = e0 + stride < n2;
    double2 aq[2], au[2], vv[2][CH];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long e = e0 + h * stride;
      const bool ok = h == 0 || two;
      if (first) {
        // V_j is read before it is overwritten by q_j (same thread, same element)
        const double2 vj = ok ? q2[e] : make_double2(0.0, 0.0);
        const double2 ww = ok ? __ldg(w2 + e) : make_double2(0.0, 0.0);
        aq[h] = make_double2(cqj * vj.x, cqj * vj.y);
        au[h] = make_double2(fma(cuj, vj.x, ww.x), fma(cuj, vj.y, ww.y));
      } else {
        aq[h] = (wq && ok) ? q2[e] : make_double2(0.0, 0.0);
        au[h] = ok ? u2[e] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int l = 0; l < CH; ++l)
        if (l < cnt) vv[h][l] = ok ? __ldg(reinterpret_cast<const double2*>(b.V[i0 + l]) + e) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long long e = e0 + h * stride;
#pragma unroll
      for (int l = 0; l < CH; ++l) {
        if (l < cnt) {
          aq[h].x = fma(cq[l], vv[h][l].x, aq[h].x);
          aq[h].y = fma(cq[l], vv[h][l].y, aq[h].y);
          au[h].x = fma(cu[l], vv[h][l].x, au[h].x);
          au[h].y = fma(cu[l], vv[h][l].y, au[h].y);
        }
      }
      if (h == 0 || two) {
        if (wq) q2[e] = aq[h];
        u2[e] = au[h];
        if (last) acc[0] = fma(au[h].x, au[h].x, fma(au[h].y, au[h].y, acc[0]));
      }
    }
  }
  if (last) block_reduce_store<1>(acc, 1, partial, nullptr);
}

// apply the stored rotations 0..j-1 to the column col[0..j+1], then form rotation j; returns the
// rotated column in R's column j and updates g from gsave[j] (g_j before the rotation)
// (csr / snr: the stored rotations 0..j-1, staged in shared memory by the caller -- a serial chain of
// global loads on one thread was most of the finishing kernels' 8-15 us)
__device__ void dcgs_rotate_column(GmresState* st, double* col, int j, const double* csr, const double* snr) {
  double* R = st->H;
  for (int i = 0; i < j; ++i) {
    const double a = col[i], b = col[i + 1];
    col[i] = csr[i] * a + snr[i] * b;
    col[i + 1] = -snr[i] * a + csr[i] * b;
  }
  const double a = col[j], b = col[j + 1];
  const double den = hypot(a, b);
  st->cs[j] = den > 0.0 ? a / den : 1.0;
  st->sn[j] = den > 0.0 ? b / den : 0.0;
  for (int i = 0; i < j; ++i) R[i + j * kLdH] = col[i];
  R[j + j * kLdH] = den;
  R[(j + 1) + j * kLdH] = 0.0;
  const double gj = st->gsave[j];
  st->g[j + 1] = -st->sn[j] * gj;
  st->g[j] = st->cs[j] * gj;
}

__global__ void __launch_bounds__(256) dcgs_finish_a_kernel(GmresState* st, const double* __restrict__ partial,
                                                            int nblk, int j, double* vscale, const int* skip) {
  if (skip_launch(skip)) return;
  __shared__ double red[2 * 52 + 2];
  // rows 0..j of the raw Hessenberg columns 0..j-1, the basis scales and the stored rotations, staged by
  // all threads: thread 0's serial algebra below then reads shared memory only
  __shared__ double sH[kLdH * 51], svs[52], scs[52], ssn[52];
  for (int e = threadIdx.x; e < j * kLdH; e += blockDim.x)
    if (e % kLdH <= j) sH[e] = st->Hraw[e];
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    svs[i] = vscale[i];
    scs[i] = st->cs[i];
    ssn[i] = st->sn[i];
  }
  const int NT = 2 * j + 2;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int t = wp; t < NT; t += (int)(blockDim.x >> 5)) {
    double v = 0.0;
    for (int bb = lane; bb < nblk; bb += 32) v += partial[(long long)bb * NT + t];
    v = warp_sum(v);
    if (lane == 0) red[t] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double* Hr = st->Hraw;
  const double sj = svs[j];
  if (j == 0) {
    // q_0 = s_0 V_0 is exactly normalised (explicit norm of r_0): one CGS pass, nu = 1
    const double gam = red[1] * sj;
    Hr[0] = gam;
    st->cu[0] = -gam * sj;
    st->cq[0] = 0.0;
    st->nu = 1.0;
    return;
  }
  double a[52], c[52], t[52], qtw[52];
  double ss = 0.0, sc = 0.0;
  for (int i = 0; i < j; ++i) {
    a[i] = red[i] * svs[i] * sj;
    c[i] = red[j + i] * svs[i];
    ss += a[i] * a[i];
    sc += a[i] * c[i];
  }
  const double sig = red[2 * j] * sj * sj, gam = red[2 * j + 1] * sj;
  const double nu2 = sig - ss;  // ||u - Q a||^2 by Pythagoras (u once-orthogonalised: a = O(eps))
  const double nu = nu2 > 0.0 ? sqrt(nu2) : 0.0;
  st->nu = nu;
  // column j-1: K q_{j-1} = Q_{j-1} h + nu1 u  and  u = Q_{j-1} a + nu q_j
  const double nu1 = sH[j + (j - 1) * kLdH];
  double col[53];
  for (int i = 0; i < j; ++i) {
    const double h = sH[i + (j - 1) * kLdH] + nu1 * a[i];
    sH[i + (j - 1) * kLdH] = h;
    Hr[i + (j - 1) * kLdH] = h;
    col[i] = h;
  }
  sH[j + (j - 1) * kLdH] = nu1 * nu;
  Hr[j + (j - 1) * kLdH] = nu1 * nu;
  col[j] = nu1 * nu;
  dcgs_rotate_column(st, col, j - 1, scs, ssn);
  if (nu == 0.0) {
    // u_j lies in span(Q_{j-1}): column j-1 was exact (lucky breakdown); the update pass becomes a
    // no-op on V_j and finish_b is skipped; the y solve uses the j corrected columns
    st->breakdown = 1;
    st->converged = 1;
    st->kcols = j;
    st->relres = fabs(st->g[j]) / st->beta0;
    for (int i = 0; i <= j; ++i) st->cq[i] = st->cu[i] = 0.0;
    st->cq[j] = 1.0;
    return;
  }
  // K q_j = (w - Q_j t)/nu with t = Hbar_{0..j, 0..j-1} a  (K Q_{j-1} = Q_j Hbar)
  for (int l = 0; l <= j; ++l) {
    double v = 0.0;
    for (int i = (l > 0 ? l - 1 : 0); i < j; ++i) v += sH[l + i * kLdH] * a[i];
    t[l] = v;
  }
  for (int i = 0; i < j; ++i) qtw[i] = c[i];
  qtw[j] = (gam - sc) / nu;  // q_j . w
  for (int l = 0; l <= j; ++l) Hr[l + j * kLdH] = (qtw[l] - t[l]) / nu;  // tentative column j
  // q_j = (s_j V_j - sum_i a_i s_i V_i)/nu;  nu u_{j+1} = w - (qtw_j/nu) u - sum_i (c_i - qtw_j a_i/nu) q_i
  const double ej = qtw[j] / nu;
  for (int i = 0; i < j; ++i) {
    st->cq[i] = -a[i] * svs[i] / nu;
    st->cu[i] = -(c[i] - ej * a[i]) * svs[i];
  }
  st->cq[j] = sj / nu;
  st->cu[j] = -ej * sj;
  vscale[j] = 1.0;  // V_j holds q_j after the update pass (which reads cq/cu only)
}

__global__ void __launch_bounds__(256) dcgs_finish_b_kernel(GmresState* st, const double* __restrict__ pnrm, int nblk,
                                                            int j, double tol, double* vscale, const int* skip,
                                                            GraphCond gc) {
  if (skip_launch(skip)) {  // (uniform over the block, before the reduction's barriers)
    // lucky breakdown in finish_a: stop the captured cycle with finish_a's column count
    if (gc.on && threadIdx.x == 0) {
      st->steps = j + 1;
      if (gc.h_cont) cudaGraphSetConditional(gc.h_cont, 0u);
    }
    return;
  }
  // column j of the raw Hessenberg matrix and the stored rotations, staged by all threads (see finish_a)
  __shared__ double scol[53], scs[52], ssn[52];
  for (int i = threadIdx.x; i <= j; i += blockDim.x) {
    scol[i] = st->Hraw[i + j * kLdH];
    scs[i] = st->cs[i];
    ssn[i] = st->sn[i];
  }
  const double nrm2 = block_sum_partials(pnrm, nblk);  // (its barriers also publish the staged values)
  if (threadIdx.x != 0) return;
  double* Hr = st->Hraw;
  const double un = sqrt(nrm2);
  const double nu = st->nu;
  Hr[(j + 1) + j * kLdH] = un / nu;  // ||u_{j+1}|| (u' = nu u_{j+1})
  vscale[j + 1] = un > 0.0 ? 1.0 / un : 0.0;
  double col[53];
  for (int i = 0; i <= j; ++i) col[i] = scol[i];
  col[j + 1] = un / nu;
  st->gsave[j] = st->g[j];
  dcgs_rotate_column(st, col, j, scs, ssn);
  st->relres = fabs(st->g[j + 1]) / st->beta0;
  st->converged = st->relres <= tol ? 1 : 0;
  st->breakdown = (un == 0.0) ? 1 : 0;
  st->kcols = j + 1;
  if (gc.on) {
    st->steps = j + 1;
    if (gc.h_cont) cudaGraphSetConditional(gc.h_cont, (st->converged | st->breakdown) ? 0u : 1u);
  }
}

// dense [rows][n_d] <-> padded [rows][P]
__global__ void pack_kernel(const double* __restrict__ dense, double* __restrict__ padded, long long rows, int nd, int P) {
  const long long total = rows * P;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / P;
    const int c = (int)(e % P);
    padded[e] = c < nd ? dense[r * nd + c] : 0.0;
  }
}

__global__ void unpack_kernel(const double* __restrict__ padded, double* __restrict__ dense, long long rows, int nd, int P) {
  const long long total = rows * nd;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / nd;
    const int c = (int)(e % nd);
    dense[e] = padded[r * P + c];
  }
}

// max/min of e over interior grid x M half levels
__global__ void __launch_bounds__(256) emaxmin_kernel(ECoef e, const double* __restrict__ a_half,
                                                      const double* __restrict__ b_half, int M, int grid_static,
                                                      Geom geo, double* partial) {
  const long long N = (long long)geo.n[0] * geo.n[1] * geo.n[2];
  double mx = -INFINITY, mn = INFINITY;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < N * M; t += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(t / N);
    const long long idx = t % N;
    double val;
    if (e.kind == 2) {
      val = e.grid[(grid_static ? 0 : (long long)m * N) + idx];
    } else {
      int c[3];
      c[2] = (int)(idx % geo.n[2]);
      c[1] = (int)((idx / geo.n[2]) % geo.n[1]);
      c[0] = (int)(idx / ((long long)geo.n[2] * geo.n[1]));
      double prod = 1.0, sum = 0.0;
      for (int i = 0; i < geo.d; ++i) {
        const int ci = c[i];  // unused trailing axes have size 1
        if (e.g[i]) prod *= e.g[i][ci];
        if (e.k[i]) sum += e.k[i][ci];
      }
      val = a_half[m] + b_half[m] * prod + sum;
    }
    mx = fmax(mx, val);
    mn = fmin(mn, val);
  }
  __shared__ double smx[8], smn[8];
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { smx[w] = mx; smn[w] = mn; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) { mx = fmax(mx, smx[k]); mn = fmin(mn, smn[k]); }
    mx = fmax(mx, smx[0]);
    mn = fmin(mn, smn[0]);
    partial[2 * blockIdx.x] = mx;
    partial[2 * blockIdx.x + 1] = mn;
  }
}

// F = (prod_l calH_{alpha_l} f)|_interior on the closed grid (Appendix; calH_l of
// Eq.(2.2)): 3^d-point stencil with weights prod_l (1 - alpha_l/12 | alpha_l/24).
__global__ void __launch_bounds__(256) compact_source_kernel(const double* __restrict__ fc, double* __restrict__ F, Geom g,
                                                             double w00, double w01, double w10, double w11,
                                                             double w20, double w21) {
  const long long N = (long long)g.n[0] * g.n[1] * g.n[2];
  const int c0 = g.n[0] + 2, c1 = g.d >= 2 ? g.n[1] + 2 : 1, c2 = g.d >= 3 ? g.n[2] + 2 : 1;
  const double w[3][2] = {{w00, w01}, {w10, w11}, {w20, w21}};
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (long long)gridDim.x * blockDim.x) {
    const int j2 = (int)(e % g.n[2]);
    const int j1 = (int)((e / g.n[2]) % g.n[1]);
    const int j0 = (int)(e / ((long long)g.n[2] * g.n[1]));
    double acc = 0.0;
    for (int a = -1; a <= 1; ++a) {
      const double wa = w[0][a != 0];
      for (int b = (g.d >= 2 ? -1 : 0); b <= (g.d >= 2 ? 1 : 0); ++b) {
        const double wb = g.d >= 2 ? w[1][b != 0] : 1.0;
        for (int cc = (g.d >= 3 ? -1 : 0); cc <= (g.d >= 3 ? 1 : 0); ++cc) {
          const double wc = g.d >= 3 ? w[2][cc != 0] : 1.0;
          long long off = (long long)(j0 + 1 + a);
          if (g.d >= 2) off = off * c1 + (j1 + 1 + b);
          if (g.d >= 3) off = off * c2 + (j2 + 1 + cc);
          acc = fma(wa * wb * wc, fc[off], acc);
        }
      }
    }
    (void)c0;
    F[e] = acc;
  }
}

// ------------------------------------------------------------------------------ launchers
static inline unsigned grid_for(long long n, int nblk) {
  long long b = (n + 255) / 256;
  if (b > nblk) b = nblk;
  if (b < 1) b = 1;
  return (unsigned)b;
}

int reduction_blocks(long long NP, int nblk) { return (int)grid_for(NP / 2, nblk); }

static BasisPtrs make_basis(const double* const* V, int J) {
  BasisPtrs b;
  for (int i = 0; i < kMaxBasis; ++i) b.V[i] = i < J ? V[i] : nullptr;
  return b;
}

// the <<<>>> argument list cannot be split by a macro comma, so use explicit wrappers
template <int JP>
static void run_dots(unsigned g, cudaStream_t s, BasisPtrs b, const double* vs, int J, const double* z, double* part,
                     long long n2) {
  dots_kernel<JP><<<g, 256, 0, s>>>(b, vs, J, z, part, n2);
}
template <int JP>
static void run_dots_upd(unsigned g, cudaStream_t s, BasisPtrs b, const double* vs, int J, const double* z,
                         const double* c, double* part, long long n) {
  dots_after_update_kernel<JP><<<g, 256, 0, s>>>(b, vs, J, z, c, part, n);
}
template <int JP>
static void run_upd_norm(unsigned g, cudaStream_t s, BasisPtrs b, const double* vs, int J, const double* z,
                         const double* c1, const double* c2, double* out, double* part, long long n2) {
  update_norm_kernel<JP><<<g, 256, 0, s>>>(b, vs, J, z, c1, c2, out, part, n2);
}
template <int JP>
static void run_axpy(unsigned g, cudaStream_t s, BasisPtrs b, const double* vs, int J, const double* y, double* x,
                     long long n2) {
  axpy_basis_kernel<JP><<<g, 256, 0, s>>>(b, vs, J, y, x, n2);
}

#define RSFDE_JP(FN, J, ...)                         \
  do {                                               \
    if ((J) <= 4) FN<4>(__VA_ARGS__);                \
    else if ((J) <= 8) FN<8>(__VA_ARGS__);           \
    else if ((J) <= 12) FN<12>(__VA_ARGS__);         \
    else if ((J) <= 16) FN<16>(__VA_ARGS__);         \
    else if ((J) <= 24) FN<24>(__VA_ARGS__);         \
    else if ((J) <= 32) FN<32>(__VA_ARGS__);         \
    else if ((J) <= 40) FN<40>(__VA_ARGS__);         \
    else FN<52>(__VA_ARGS__);                        \
  } while (0)

cudaError_t launch_dots(const double* const* V, const double* vscale, int J, const double* z, double* partial,
                        long long NP, int nblk, cudaStream_t s) {
  if (J < 1 || J > kMaxBasis) return cudaErrorInvalidValue;
  const unsigned g = grid_for(NP / 2, nblk);
  RSFDE_JP(run_dots, J, g, s, make_basis(V, J), vscale, J, z, partial, NP / 2);
  return cudaGetLastError();
}

cudaError_t launch_dots_after_update(const double* const* V, const double* vscale, int J, const double* z,
                                     const double* coef, double* partial, long long NP, int nblk, cudaStream_t s) {
  if (J < 1 || J > kMaxBasis) return cudaErrorInvalidValue;
  const unsigned g = grid_for(NP / 2, nblk);  // same block count as the other reductions
  RSFDE_JP(run_dots_upd, J, g, s, make_basis(V, J), vscale, J, z, coef, partial, NP / 2);
  return cudaGetLastError();
}

cudaError_t launch_update_norm(const double* const* V, const double* vscale, int J, const double* z, const double* c1,
                               const double* c2, double* out, double* partial, long long NP, int nblk, cudaStream_t s) {
  if (J < 1 || J > kMaxBasis) return cudaErrorInvalidValue;
  const unsigned g = grid_for(NP / 2, nblk);
  RSFDE_JP(run_upd_norm, J, g, s, make_basis(V, J), vscale, J, z, c1, c2, out, partial, NP / 2);
  return cudaGetLastError();
}

cudaError_t launch_axpy_basis(const double* const* V, const double* vscale, int J, const double* y, double* x,
                              long long NP, cudaStream_t s) {
  if (J < 1 || J > kMaxBasis) return cudaErrorInvalidValue;
  const unsigned g = grid_for(NP / 2, stream_blocks());
  RSFDE_JP(run_axpy, J, g, s, make_basis(V, J), vscale, J, y, x, NP / 2);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double* partial, int nblk, int J, double* out, cudaStream_t s) {
  reduce_kernel<<<1, 256, 0, s>>>(partial, nblk, J, out);
  return cudaGetLastError();
}

cudaError_t launch_sumsq(const double* z, double* partial, long long NP, int nblk, cudaStream_t s) {
  sumsq_kernel<<<grid_for(NP / 2, nblk), 256, 0, s>>>(z, partial, NP / 2);
  return cudaGetLastError();
}

cudaError_t launch_axpby(double a, const double* x, double b, double* y, long long NP, cudaStream_t s) {
  axpby_kernel<<<grid_for(NP / 2, stream_blocks()), 256, 0, s>>>(a, x, b, y, NP / 2);
  return cudaGetLastError();
}

cudaError_t launch_pack(const double* dense, double* padded, const Geom& g, cudaStream_t s) {
  const long long rows = g.NP / g.P;
  pack_kernel<<<grid_for(g.NP, stream_blocks()), 256, 0, s>>>(dense, padded, rows, g.n[g.d - 1], g.P);
  return cudaGetLastError();
}

cudaError_t launch_unpack(const double* padded, double* dense, const Geom& g, cudaStream_t s) {
  const long long rows = g.NP / g.P;
  unpack_kernel<<<grid_for(rows * g.n[g.d - 1], stream_blocks()), 256, 0, s>>>(padded, dense, rows, g.n[g.d - 1], g.P);
  return cudaGetLastError();
}

cudaError_t launch_compact_source(const double* f_closed, double* F, const Geom& g, const double* alpha,
                                  cudaStream_t s) {
  double w[3][2];
  for (int i = 0; i < 3; ++i) {
    w[i][0] = 1.0 - alpha[i] / 12.0;
    w[i][1] = alpha[i] / 24.0;
  }
  const long long N = (long long)g.n[0] * g.n[1] * g.n[2];
  compact_source_kernel<<<grid_for(N, stream_blocks()), 256, 0, s>>>(f_closed, F, g, w[0][0], w[0][1], w[1][0], w[1][1],
                                                              w[2][0], w[2][1]);
  return cudaGetLastError();
}

cudaError_t launch_emaxmin(const ECoef& e, const double* a_half, const double* b_half, int M, int grid_static,
                           const Geom& geo, double* partial, int nblk, cudaStream_t s) {
  emaxmin_kernel<<<nblk, 256, 0, s>>>(e, a_half, b_half, M, grid_static, geo, partial);
  return cudaGetLastError();
}

cudaError_t launch_arnoldi_finish(GmresState* st, const double* h1, const double* h2, const double* partial_nrm,
                                  int nblk, int j, double tol, double* vscale_next, cudaStream_t s) {
  arnoldi_finish_kernel<<<1, 256, 0, s>>>(st, h1, h2, partial_nrm, nblk, j, tol, vscale_next);
  return cudaGetLastError();
}

cudaError_t launch_gmres_init(GmresState* st, const double* partial_nrm, int nblk, double* vscale0, int first_cycle,
                              cudaStream_t s, GraphCond gc) {
  gmres_init_kernel<<<1, 256, 0, s>>>(st, partial_nrm, nblk, vscale0, first_cycle, gc);
  return cudaGetLastError();
}

template <int CH>
static void run_dcgs_dots(unsigned g, cudaStream_t s, BasisPtrs b, int i0, int cnt, int j, int first, const double* w,
                          double* part, int NT, long long n2, const int* skip) {
  dcgs_dots_kernel<CH><<<g, 256, 0, s>>>(b, i0, cnt, j, first, w, part, NT, n2, skip);
}
template <int CH>
static void run_dcgs_update(unsigned g, cudaStream_t s, BasisPtrs b, int i0, int cnt, int j, int first, int last,
                            const GmresState* st, const double* w, double* oq, double* ou, double* part,
                            long long n2, const int* skip) {
  dcgs_update_kernel<CH><<<g, 256, 0, s>>>(b, i0, cnt, j, first, last, st, w, oq, ou, part, n2, skip);
}
#define RSFDE_CH(FN, C, ...)                 \
  do {                                       \
    if ((C) <= 2) FN<2>(__VA_ARGS__);        \
    else if ((C) <= 4) FN<4>(__VA_ARGS__);   \
    else FN<8>(__VA_ARGS__);                 \
  } while (0)

// basis vectors per dots / update launch: at most 8 keeps a thread (two elements in flight) within 128
// registers, two 256-thread blocks per SM; longer bases take several launches (u and w re-read)
constexpr int kDcgsChunk = 8;

cudaError_t launch_dcgs_dots(const double* const* V, int j, const double* w, double* partial, long long NP, int nblk,
                             const int* skip, cudaStream_t s) {
  if (j < 0 || j + 1 >= kMaxBasis) return cudaErrorInvalidValue;
  const unsigned g = grid_for(NP / 2, nblk);
  const BasisPtrs b = make_basis(V, j + 1);
  const int NT = 2 * j + 2;
  // chunks of <= kDcgsChunk basis vectors (u and w are re-read per extra chunk)
  for (int i0 = 0; i0 == 0 || i0 < j; i0 += kDcgsChunk) {
    const int cnt = j - i0 < kDcgsChunk ? j - i0 : kDcgsChunk;
    RSFDE_CH(run_dcgs_dots, cnt, g, s, b, i0, cnt, j, i0 == 0 ? 1 : 0, w, partial, NT, NP / 2, skip);
  }
  return cudaGetLastError();
}

cudaError_t launch_dcgs_finish_a(GmresState* st, const double* partial, int nblk, int j, double* vscale, const int* skip,
                                 cudaStream_t s) {
  dcgs_finish_a_kernel<<<1, 256, 0, s>>>(st, partial, nblk, j, vscale, skip);
  return cudaGetLastError();
}

cudaError_t launch_dcgs_update(const double* const* V, int j, const GmresState* st, const double* w,
                               double* partial_nrm, long long NP, int nblk, const int* skip, cudaStream_t s) {
  if (j < 0 || j + 2 > kMaxBasis) return cudaErrorInvalidValue;
  const unsigned g = grid_for(NP / 2, nblk);
  const BasisPtrs b = make_basis(V, j + 2);
  double* oq = const_cast<double*>(V[j]);
  double* ou = const_cast<double*>(V[j + 1]);
  for (int i0 = 0; i0 == 0 || i0 < j; i0 += kDcgsChunk) {
    const int cnt = j - i0 < kDcgsChunk ? j - i0 : kDcgsChunk;
    const int last = i0 + kDcgsChunk >= j ? 1 : 0;
    RSFDE_CH(run_dcgs_update, cnt, g, s, b, i0, cnt, j, i0 == 0 ? 1 : 0, last, st, w, oq, ou, partial_nrm, NP / 2, skip);
  }
  return cudaGetLastError();
}

cudaError_t launch_dcgs_finish_b(GmresState* st, const double* partial_nrm, int nblk, int j, double tol, double* vscale,
                                 const int* skip, cudaStream_t s, GraphCond gc) {
  dcgs_finish_b_kernel<<<1, 256, 0, s>>>(st, partial_nrm, nblk, j, tol, vscale, skip, gc);
  return cudaGetLastError();
}

cudaError_t launch_gmres_solve_y(GmresState* st, int k, cudaStream_t s) {
  gmres_solve_y_kernel<<<1, 32, 0, s>>>(st, k);
  return cudaGetLastError();
}

// SWITCH selector of a captured cycle: the column count of the y solve (kcols < 0: r0 == 0, none)
__global__ void graph_set_k_kernel(const GmresState* st, unsigned long long hk) {
  cudaGraphSetConditional(hk, st->kcols > 0 ? (unsigned)st->kcols : 0u);
}
cudaError_t launch_graph_set_k(const GmresState* st, unsigned long long hk, cudaStream_t s) {
  graph_set_k_kernel<<<1, 1, 0, s>>>(st, hk);
  return cudaGetLastError();
}

__global__ void set_ab_kernel(double* ab, double a, double b) {
  ab[0] = a;
  ab[1] = b;
}
cudaError_t launch_set_ab(double* ab, double a, double b, cudaStream_t s) {
  set_ab_kernel<<<1, 1, 0, s>>>(ab, a, b);
  return cudaGetLastError();
}

}  // namespace rsfde
