// Single-CTA blocked Householder QR for the sweep-sized unfoldings (m x n up to ~27 K doubles
// in shared memory): panels of 16 columns factored column by column (one warp per trailing
// panel column, LAPACK dlarfg signs), the dlarft T factor, and the compact-WY trailing update
// Y = V^T A2, Z = T^T Y, A2 -= V Z on the DMMA pipe (mma.m8n8k4.f64); Q formed in place as
// dorgqr does (block reflectors applied backwards, dorg2r inside each panel).  Same reflectors
// and signs as the unblocked kernel (linalg.cu qr_kernel) -- Q and R match numpy.linalg.qr --
// but the trailing matrix is read once per panel instead of once per column.
#include <algorithm>

#include "dmma_tile.cuh"
#include "linalg.cuh"

namespace qtt {
namespace {

constexpr int QNT = 512;  // 16 warps
constexpr int QNW = QNT / 32;
constexpr int BP = 16;    // panel width

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct QrSmem {
  double* W;    // ldm x n, column-major
  double* tau;  // k
  double* T;    // BP x BP (row-major, upper triangular)
  double* Y;    // BP x n  (row-major, ld n)
  int ldm;
};

// V[i][r] of the panel starting at column p0 (unit lower trapezoidal, reflectors below the diagonal)
__device__ __forceinline__ double vval(const QrSmem& s, int m, int p0, int bp, int i, int r) {
  const int j = p0 + r;
  if (r >= bp || i < j || i >= m) return 0.0;
  return i == j ? 1.0 : s.W[i + (long long)j * s.ldm];
}

// Y[r][c - c0] = sum_{i >= p0} V[i][r] W[i][c] for c in [c0, c1)  (DMMA: M = 16, N = c1 - c0,
// K = m - p0).  The K range is split in two halves -- the first summed into Y, the second into
// Y2 -- and each half runs two independent accumulator chains (even / odd k-steps).
__device__ void panel_vt_a(const QrSmem& s, int m, int p0, int bp, int c0, int c1, double* Y2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int nt = c1 - c0;
  const int FN = (nt + 7) / 8, F = 2 * FN;
  const int K = m - p0, kh = ((K + 15) / 16) * 8;  // half of K, a multiple of 8
  for (int item = warp; item < 2 * F; item += QNW) {
    const int f = item >> 1, half = item & 1;
    const int fr = f / FN, fc = f - fr * FN;
    double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0};
    const int r = fr * 8 + lr;        // A fragment row (V column)
    const int cb = c0 + fc * 8 + lr;  // B fragment column
    const int kb = p0 + half * kh, ke = min(m, kb + kh);
    for (int k = kb; k < ke; k += 8) {
      const int i = k + lc, i2 = k + 4 + lc;
      const double x0 = vval(s, m, p0, bp, i, r), x1 = vval(s, m, p0, bp, i2, r);
      const double y0 = (i < m && cb < c1) ? s.W[i + (long long)cb * s.ldm] : 0.0;
      const double y1 = (i2 < m && cb < c1) ? s.W[i2 + (long long)cb * s.ldm] : 0.0;
      tile::dmma(a0, x0, y0);
      tile::dmma(a1, x1, y1);
    }
    double* out = half ? Y2 : s.Y;
    const int row = fr * 8 + lr, col = fc * 8 + lc * 2;
    if (col < nt) out[row * nt + col] = a0[0] + a1[0];
    if (col + 1 < nt) out[row * nt + col + 1] = a0[1] + a1[1];
  }
}

// Y <- -op(T) (Y + Y2) (op = T^T when trans, else T); Y, Y2 are BP x nt row-major, nt <= 256
__device__ void apply_t(const QrSmem& s, int bp, int nt, bool trans, const double* Y2) {
  constexpr int PER = (BP * 256 + QNT - 1) / QNT;
  double out[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * QNT;
    double v = 0.0;
    if (e < BP * nt) {
      const int r = e / nt, c = e - r * nt;
      if (r < bp) {
        if (trans)
          for (int q = 0; q <= r; ++q) v += s.T[q * BP + r] * (s.Y[q * nt + c] + Y2[q * nt + c]);
        else
          for (int q = r; q < bp; ++q) v += s.T[r * BP + q] * (s.Y[q * nt + c] + Y2[q * nt + c]);
      }
    }
    out[u] = -v;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int e = threadIdx.x + u * QNT;
    if (e < BP * nt) s.Y[e] = out[u];
  }
  __syncthreads();
}

// W[i][c] += sum_r V[i][r] Y[r][c - c0] for i in [p0, m), c in [c0, c1)   (Y holds -Z); two
// fragments per warp pass, so their DMMA chains overlap
__device__ void panel_update(const QrSmem& s, int m, int p0, int bp, int c0, int c1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int nt = c1 - c0;
  const int FM = (m - p0 + 7) / 8, FN = (nt + 7) / 8, F = FM * FN;
  for (int f0 = warp; f0 < F; f0 += 2 * QNW) {
    double acc[2][2];
    int crow[2], ccol[2], i0[2], fn[2];
    bool on[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int f = f0 + u * QNW;
      on[u] = f < F;
      const int fm = on[u] ? f / FN : 0;
      fn[u] = on[u] ? f - fm * FN : 0;
      i0[u] = p0 + fm * 8;
      crow[u] = i0[u] + lr;
      ccol[u] = c0 + fn[u] * 8 + lc * 2;
      acc[u][0] = (on[u] && crow[u] < m && ccol[u] < c1) ? s.W[crow[u] + (long long)ccol[u] * s.ldm] : 0.0;
      acc[u][1] = (on[u] && crow[u] < m && ccol[u] + 1 < c1) ? s.W[crow[u] + (long long)(ccol[u] + 1) * s.ldm] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < BP; k += 4) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const double a = vval(s, m, p0, bp, i0[u] + lr, k + lc);
        const int bc = fn[u] * 8 + lr;
        const double b = bc < nt ? s.Y[(k + lc) * nt + bc] : 0.0;
        tile::dmma(acc[u], a, b);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (on[u] && crow[u] < m) {
        if (ccol[u] < c1) s.W[crow[u] + (long long)ccol[u] * s.ldm] = acc[u][0];
        if (ccol[u] + 1 < c1) s.W[crow[u] + (long long)(ccol[u] + 1) * s.ldm] = acc[u][1];
      }
    }
  }
}

// apply reflector j (v in column j below the diagonal, tau[j]) to column c, rows j..m-1 (one warp).
// The lane's MPL rows (i = lane + 32 t) are loaded together, so the dot and the update each cost
// one shared-memory round trip instead of one per 32 rows.
template <int MPL>
__device__ __forceinline__ void reflect_col(const QrSmem& s, int m, int j, int c, double t) {
  const int lane = threadIdx.x & 31;
  const double* vj = s.W + (long long)j * s.ldm;
  double* wc = s.W + (long long)c * s.ldm;
  double v[MPL], x[MPL];
  double w = 0.0;
#pragma unroll
  for (int u = 0; u < MPL; ++u) {
    const int i = lane + 32 * u;
    const bool in = i > j && i < m;
    v[u] = in ? vj[i] : 0.0;
    x[u] = in ? wc[i] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < MPL; ++u) w = fma(v[u], x[u], w);
  w = (wsum(w) + wc[j]) * t;
  if (lane == 0) wc[j] -= w;
#pragma unroll
  for (int u = 0; u < MPL; ++u) {
    const int i = lane + 32 * u;
    if (i > j && i < m) wc[i] = fma(-w, v[u], x[u]);
  }
}

// sum_{i > j} W[i][j]^2 over one warp (the same register-batched loads)
template <int MPL>
__device__ __forceinline__ double col_norm2(const QrSmem& s, int m, int j) {
  const int lane = threadIdx.x & 31;
  const double* vj = s.W + (long long)j * s.ldm;
  double x[MPL], part = 0.0;
#pragma unroll
  for (int u = 0; u < MPL; ++u) {
    const int i = lane + 32 * u;
    x[u] = (i > j && i < m) ? vj[i] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < MPL; ++u) part = fma(x[u], x[u], part);
  return wsum(part);
}

// T of the panel (dlarft, forward columnwise: T[0:i, i] = -tau_i T[0:i, 0:i] (V[:, 0:i]^T v_i)).
// G = V^T V on the DMMA pipe (4 warps per 8x8 block, K split 4 ways, fixed-order sum), then the
// triangular recursion by warp 0 (lane q owns row q).  Ends with a block barrier.
__device__ void build_t(const QrSmem& s, int m, int p0, int bp, double* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  {
    const int f = warp & 3, part = warp >> 2;  // fragment (2x2 blocks of 8) and K quarter
    const int fr = f >> 1, fc = f & 1;
    const int K = m - p0, kq = ((K + 15) / 16) * 4;
    const int kb = p0 + part * kq, ke = min(m, kb + kq);
    double acc[2] = {0.0, 0.0};
    for (int k = kb; k < ke; k += 4) {
      const int i = k + lc;
      tile::dmma(acc, vval(s, m, p0, bp, i, fr * 8 + lr), vval(s, m, p0, bp, i, fc * 8 + lr));
    }
    double* P = tmp + part * BP * BP;
    const int row = fr * 8 + lr, col = fc * 8 + lc * 2;
    P[row * BP + col] = acc[0];
    P[row * BP + col + 1] = acc[1];
  }
  __syncthreads();
  // G = the four K quarters summed in order (all threads), then the recursion
  double* G = tmp + 4 * BP * BP;
  for (int e = threadIdx.x; e < BP * BP; e += QNT)
    G[e] = ((tmp[e] + tmp[BP * BP + e]) + tmp[2 * BP * BP + e]) + tmp[3 * BP * BP + e];
  __syncthreads();
  if (warp == 0) {
    const int q = lane;
    double trow[BP];
#pragma unroll
    for (int u = 0; u < BP; ++u) trow[u] = 0.0;
#pragma unroll
    for (int i = 0; i < BP; ++i) {
      if (i < bp) {
        double g[BP];
#pragma unroll
        for (int u = 0; u < BP; ++u) g[u] = (u < i) ? G[u * BP + i] : 0.0;  // loads in flight together
        const double ti = s.tau[p0 + i];
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < BP; ++u)
          if (u < i && u >= q) v = fma(trow[u], g[u], v);
        trow[i] = q < i ? -ti * v : (q == i ? ti : 0.0);  // row q of T gains column i
      }
    }
    if (q < BP)
#pragma unroll
      for (int u = 0; u < BP; ++u) s.T[q * BP + u] = q < bp ? trow[u] : 0.0;
  }
  __syncthreads();
}

// dlarfg (LAPACK sign rule) of a column with pivot alpha and sum of squares xnorm2 below it:
// dst = {tau, beta, 1 / (alpha - beta), xnorm2}
__device__ __forceinline__ void dlarfg_to(double alpha, double xnorm2, double* dst) {
  double t = 0.0, beta = alpha, scal = 1.0;
  if (xnorm2 > 0.0) {
    beta = -copysign(hypot(alpha, sqrt(xnorm2)), alpha);
    t = (beta - alpha) / beta;
    scal = 1.0 / (alpha - beta);
  }
  dst[0] = t;
  dst[1] = beta;
  dst[2] = scal;
  dst[3] = xnorm2;
}

// reflect_col with the reflector still unscaled in shared memory (v = x * scal formed on the fly:
// the same product as scaling in place, so the same bits).  With next != nullptr (the warp owning
// the next pivot column, c == j + 1) the updated column's dlarfg is computed here, from registers.
template <int MPL>
__device__ __forceinline__ void reflect_col_s(const QrSmem& s, int m, int j, int c, double t, double scal,
                                              double* next) {
  const int lane = threadIdx.x & 31;
  const double* vj = s.W + (long long)j * s.ldm;
  double* wc = s.W + (long long)c * s.ldm;
  double v[MPL], x[MPL];
  double w = 0.0;
#pragma unroll
  for (int u = 0; u < MPL; ++u) {
    const int i = lane + 32 * u;
    const bool in = i > j && i < m;
    v[u] = in ? vj[i] * scal : 0.0;
    x[u] = in ? wc[i] : 0.0;
  }
#pragma unroll
  for (int u = 0; u < MPL; ++u) w = fma(v[u], x[u], w);
  w = (wsum(w) + wc[j]) * t;
  if (lane == 0) wc[j] -= w;
  double part = 0.0, alpha = 0.0;
#pragma unroll
  for (int u = 0; u < MPL; ++u) {
    const int i = lane + 32 * u;
    if (i > j && i < m) {
      x[u] = fma(-w, v[u], x[u]);
      wc[i] = x[u];
      if (i > c) part = fma(x[u], x[u], part);
      if (i == c) alpha = x[u];
    }
  }
  if (next != nullptr) {
    part = wsum(part);
    alpha = wsum(alpha);  // exactly one lane holds a nonzero alpha slot (the others add 0)
    if (lane == 0) dlarfg_to(alpha, part, next);
  }
}

template <int MPL>
__global__ void __launch_bounds__(QNT) qr_cta_kernel(CMatView in, MatView Qo, MatView Ro, int ldm) {
  extern __shared__ double sm[];
  __shared__ double sh[8];
  const int m = in.rows, n = in.cols, k = min(m, n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  QrSmem s;
  s.ldm = ldm;
  s.W = sm;
  s.tau = s.W + (long long)ldm * n;
  s.T = s.tau + ((k + 1) & ~1);
  s.Y = s.T + BP * BP;
  double* tmp = s.Y + BP * n;

  for (int j = warp; j < n; j += QNW)  // (row-major sources read one row per lane: a column per warp)
    for (int i = lane; i < m; i += 32) s.W[i + (long long)j * ldm] = in.p[i * in.rs + j * in.cs];
  __syncthreads();

  // ---- factor: panels of BP columns.  One block barrier per column: the reflector of column j
  // stays unscaled while the other columns read it (scaled on the fly) and is scaled in place one
  // step later by the otherwise idle last warp; the next pivot's dlarfg is computed by warp 0
  // right after it updates that column (double-buffered in sh).
  for (int p0 = 0; p0 < k; p0 += BP) {
    const int bp = min(BP, k - p0);
    if (warp == 0) {
      const double xnorm2 = col_norm2<MPL>(s, m, p0);
      if (lane == 0) dlarfg_to(s.W[p0 + (long long)p0 * ldm], xnorm2, sh);
    }
    __syncthreads();
    double prev_scal = 1.0, prev_xn = 0.0;
    for (int j = p0; j < p0 + bp; ++j) {
      double* vj = s.W + (long long)j * ldm;
      const double* cur = sh + 4 * ((j - p0) & 1);
      double* nxt = sh + 4 * ((j - p0 + 1) & 1);
      const double t = cur[0], beta = cur[1], scal = cur[2], xn = cur[3];
      if (tid == 0) {
        s.tau[j] = t;
        vj[j] = beta;
      }
      if (warp == QNW - 1 && j > p0 && prev_xn > 0.0) {  // deferred scaling of column j - 1
        double* vp = vj - ldm;
        for (int i = j + lane; i < m; i += 32) vp[i] *= prev_scal;
      }
      if (j + 1 < p0 + bp) {
        if (t != 0.0) {
          for (int c = j + 1 + warp; c < p0 + bp; c += QNW)
            reflect_col_s<MPL>(s, m, j, c, t, scal, c == j + 1 ? nxt : nullptr);
        } else if (warp == 0) {  // H_j = I: the next pivot column is untouched
          const double xnorm2 = col_norm2<MPL>(s, m, j + 1);
          if (lane == 0) dlarfg_to(s.W[(j + 1) + (long long)(j + 1) * ldm], xnorm2, nxt);
        }
      }
      prev_scal = scal;
      prev_xn = xn;
      __syncthreads();
    }
    if (prev_xn > 0.0) {  // the panel's last reflector
      double* vl = s.W + (long long)(p0 + bp - 1) * ldm;
      for (int i = p0 + bp + tid; i < m; i += QNT) vl[i] *= prev_scal;
    }
    __syncthreads();
    if (p0 + bp >= n) break;  // no trailing columns
    build_t(s, m, p0, bp, tmp);
    // trailing update with H^T = I - V T^T V^T
    const int c0 = p0 + bp;
    panel_vt_a(s, m, p0, bp, c0, n, tmp);
    __syncthreads();
    apply_t(s, bp, n - c0, true, tmp);
    panel_update(s, m, p0, bp, c0, n);
    __syncthreads();
  }

  if (Ro.p) {
    for (int i = warp; i < k; i += QNW)
      for (int c = lane; c < n; c += 32) Ro.p[i * Ro.rs + c * Ro.cs] = (i <= c) ? s.W[i + (long long)c * ldm] : 0.0;
  }
  if (!Qo.p) return;
  __syncthreads();

  // ---- Q (dorgqr): panels backwards; block reflector on the columns to the right, then
  // dorg2r inside the panel
  const int last = ((k - 1) / BP) * BP;
  for (int p0 = last; p0 >= 0; p0 -= BP) {
    const int bp = min(BP, k - p0);
    const int c0 = p0 + bp;
    if (c0 < k) {
      build_t(s, m, p0, bp, tmp);  // T of this panel (the factor pass reused the buffer)
      // rows p0..c0-1 of the columns right of the panel are zero in Q at this point
      for (int e = tid; e < bp * (k - c0); e += QNT) {
        const int r = e % bp, c = c0 + e / bp;
        s.W[p0 + r + (long long)c * ldm] = 0.0;
      }
      __syncthreads();
      panel_vt_a(s, m, p0, bp, c0, k, tmp);
      __syncthreads();
      apply_t(s, bp, k - c0, false, tmp);
      panel_update(s, m, p0, bp, c0, k);
      __syncthreads();
    }
    // dorg2r on the panel, one block barrier per column: column j+1 is finalised (e_j - tau v)
    // at the start of step j by warp 0, which then applies H_j to it
    for (int j = p0 + bp - 1; j >= p0; --j) {
      const double t = s.tau[j];
      if (warp == 0 && j + 1 < p0 + bp) {
        double* vf = s.W + (long long)(j + 1) * ldm;
        const double tf = s.tau[j + 1];
        for (int i = lane; i < m; i += 32) vf[i] = i > j + 1 ? vf[i] * -tf : (i == j + 1 ? 1.0 - tf : 0.0);
        __syncwarp();
      }
      if (t != 0.0)
        for (int c = j + 1 + warp; c < p0 + bp; c += QNW) reflect_col<MPL>(s, m, j, c, t);
      __syncthreads();
    }
    {
      double* vf = s.W + (long long)p0 * ldm;
      const double tf = s.tau[p0];
      for (int i = tid; i < m; i += QNT) vf[i] = i > p0 ? vf[i] * -tf : (i == p0 ? 1.0 - tf : 0.0);
    }
    __syncthreads();
  }
  if (Qo.cs == 1) {  // row-major Q: lanes along the row for coalesced stores
    for (int i = warp; i < m; i += QNW)
      for (int c = lane; c < k; c += 32) Qo.p[i * Qo.rs + c] = s.W[i + (long long)c * ldm];
  } else {
    for (int c = warp; c < k; c += QNW)
      for (int i = lane; i < m; i += 32) Qo.p[i * Qo.rs + c * Qo.cs] = s.W[i + (long long)c * ldm];
  }
}

}  // namespace

long long qr_cta_smem_doubles(int m, int n) {
  const int k = std::min(m, n);
  const int ldm = m + ((4 - m % 16) + 16) % 16;  // == 4 (mod 16): conflict-free fragment loads
  return (long long)ldm * n + ((k + 1) & ~1) + BP * BP + BP * n + std::max(BP * n, 5 * BP * BP);
}

void qr_cta(Ctx& c, CMatView in, MatView Q, MatView R) {
  const int m = in.rows, n = in.cols;
  const int ldm = m + ((4 - m % 16) + 16) % 16;
  const size_t bytes = (size_t)qr_cta_smem_doubles(m, n) * sizeof(double);
  static PerDevice<bool> attr_dev(false);
  bool& attr = attr_dev();
  if (!attr) {
    QTT_CUDA(cudaFuncSetAttribute(qr_cta_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    QTT_CUDA(cudaFuncSetAttribute(qr_cta_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    QTT_CUDA(cudaFuncSetAttribute(qr_cta_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024));
    attr = true;
  }
  if (m <= 256)
    qr_cta_kernel<8><<<1, QNT, bytes, c.stream>>>(in, Q, R, ldm);
  else if (m <= 512)
    qr_cta_kernel<16><<<1, QNT, bytes, c.stream>>>(in, Q, R, ldm);
  else
    qr_cta_kernel<32><<<1, QNT, bytes, c.stream>>>(in, Q, R, ldm);
  QTT_CHECK_LAUNCH();
}

}  // namespace qtt
