// Interface contractions as DMMA GEMM chains (see contract.cuh).
#include "contract.cuh"

#include <algorithm>

namespace qtt {
namespace {

__global__ void permute_op_core_kernel(const double* __restrict__ A, int R0, int m, int n, int R1,
                                       double* __restrict__ Ap, double* __restrict__ Aq) {
  const long long total = (long long)R0 * m * n * R1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    // e indexes A[a, mm, nn, b] in row-major order
    long long t = e;
    const int b = (int)(t % R1); t /= R1;
    const int nn = (int)(t % n); t /= n;
    const int mm = (int)(t % m); t /= m;
    const int a = (int)t;
    const double v = A[e];
    if (Ap) Ap[(((long long)mm * R1 + b) * R0 + a) * n + nn] = v;  // Ap[(m,B),(A,n)]
    if (Aq) Aq[(((long long)mm * R0 + a) * R1 + b) * n + nn] = v;  // Aq[(m,a),(A',n)], A' = b
  }
}

__global__ void transpose_rows_kernel(const double* __restrict__ in, double* __restrict__ out, long long rows,
                                      long long cols, long long ldo) {
  __shared__ double tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, c0 = (long long)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const long long r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const long long c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ldo + r] = tile[threadIdx.x][i];
  }
}

// split-K workspace a plain M x N x K product may ask for (gemm.cu plan)
long long splitk_ws(int M, int N, int K) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K;
  GemmArgs t = g;  // the same product with K-contiguous operands may take the TMA path
  t.a_rs = K; t.a_cs = 1; t.b_rs = 1; t.b_cs = K + (K & 1); t.c_rs = N; t.c_cs = 1;
  return std::max(gemm_workspace_hint(g), gemm_workspace_hint(t));
}

inline Scratch take(Scratch& sc, long long n) {
  if (n > sc.n) throw Error(QTT_ERR_ARG, "contraction scratch too small");
  Scratch out{sc.p, n};
  sc.p += n;
  sc.n -= n;
  return out;
}

}  // namespace

// out[c][r] = in[r][c] (in: rows x cols row-major; out rows = cols, pitch ldo)
void transpose_rows(const double* in, double* out, long long rows, long long cols, long long ldo, cudaStream_t s) {
  dim3 g((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32));
  transpose_rows_kernel<<<g, dim3(32, 8), 0, s>>>(in, out, rows, cols, ldo);
  QTT_CHECK_LAUNCH();
}

void permute_op_core(const double* A, int R0, int m, int n, int R1, double* Ap, double* Aq,
                     cudaStream_t s) {
  const long long total = (long long)R0 * m * n * R1;
  const int blocks = (int)std::min<long long>(cdiv(total, 256), 1024);
  permute_op_core_kernel<<<blocks, 256, 0, s>>>(A, R0, m, n, R1, Ap, Aq);
  QTT_CHECK_LAUNCH();
}

// Step 1 reads v as B^T (K = U contiguous) when the product is large enough for the TMA
// GEMM path: v is transposed into scratch first (rU x n*rV doubles, cheap next to the GEMM).
static bool step1_transposed(int rX, int Ra, int rU, int n, int rV) {
  return (double)rX * Ra * n * rV * rU >= (double)(1 << 24) && rU >= 64 && rX * Ra >= 64 && n * rV >= 32;
}

// ---------------------------------------------------------------- left environment
long long env_left_scratch(int rX, int RA, int rY, int m, int n, int RB, int rZ, int rU) {
  return (long long)rX * RA * n * rZ + (long long)rX * m * RB * rZ + (long long)(rY + 1) * n * rZ +
         std::max(splitk_ws(rX * RA, n * rZ, rY), splitk_ws(rU, RB * rZ, rX * m));
}

void env_left(const double* phi, int rX, int RA, int rY, const double* bra, int rU,
              const double* Ap, int m, int n, int RB, const double* ket, int rZ, double* out,
              Scratch sc, cudaStream_t s) {
  double* t1 = take(sc, (long long)rX * RA * n * rZ).p;  // [X][A][n][Z]
  double* t2 = take(sc, (long long)rX * m * RB * rZ).p;  // [X][m][B][Z]
  {  // t1[(X,A),(n,Z)] = phi[(X,A),Y] @ ket[Y,(n,Z)]   (ket read transposed when large: TMA path)
    GemmArgs g;
    g.M = rX * RA; g.N = n * rZ; g.K = rY;
    gemm_set_A(g, phi, rY, false);
    if (step1_transposed(rX, RA, rY, n, rZ)) {
      const long long ldt = rY + (rY & 1);
      double* kT = take(sc, ldt * n * rZ).p;  // [(n,Z)][Y]
      transpose_rows(ket, kT, rY, (long long)n * rZ, ldt, s);
      g.B = kT; g.b_rs = 1; g.b_cs = ldt;
    } else {
      gemm_set_B(g, ket, (long long)n * rZ, false);
    }
    gemm_set_C(g, t1, (long long)n * rZ);
    gemm(g, s, sc.p, sc.n);
  }
  {  // per X: t2[X][(m,B),Z] = Ap[(m,B),(A,n)] @ t1[X][(A,n),Z]
    GemmArgs g;
    g.M = m * RB; g.N = rZ; g.K = RA * n;
    gemm_set_A(g, Ap, (long long)RA * n, false);
    gemm_set_B(g, t1, rZ, false);
    g.b_bs1 = (long long)RA * n * rZ;
    gemm_set_C(g, t2, rZ);
    g.c_bs1 = (long long)m * RB * rZ;
    g.batch1 = rX;
    gemm(g, s);
  }
  {  // out[U,(B,Z)] = bra[(X,m),U]^T @ t2[(X,m),(B,Z)]
    GemmArgs g;
    g.M = rU; g.N = RB * rZ; g.K = rX * m;
    gemm_set_A(g, bra, rU, true);
    gemm_set_B(g, t2, (long long)RB * rZ, false);
    gemm_set_C(g, out, (long long)RB * rZ);
    gemm(g, s, sc.p, sc.n);
  }
}

// ---------------------------------------------------------------- right environment
long long env_right_scratch(int rX, int RA, int rZ, int m, int n, int Ra, int rY, int rB) {
  return (long long)rX * RA * n * rY + (long long)m * rX * Ra * rY +
         splitk_ws(rB, Ra * rY, m * rX);
}

void env_right(const double* phi, int rX, int RA, int rZ, const double* bra, int rB,
               const double* Aq, int m, int n, int Ra, const double* ket, int rY, double* out,
               Scratch sc, cudaStream_t s) {
  double* s1 = take(sc, (long long)rX * RA * n * rY).p;  // [X][A'][n][Y]
  double* s2 = take(sc, (long long)m * rX * Ra * rY).p;  // [m][X][a][Y]
  {  // per n: s1[(X,A'), n, Y] = phi[(X,A'),Z] @ ket[Y,n,Z]^T
    GemmArgs g;
    g.M = rX * RA; g.N = rY; g.K = rZ;
    gemm_set_A(g, phi, rZ, false);
    g.B = ket; g.b_rs = 1; g.b_cs = (long long)n * rZ; g.b_bs1 = rZ;
    g.C = s1; g.c_rs = (long long)n * rY; g.c_cs = 1; g.c_bs1 = rY;
    g.batch1 = n;
    gemm(g, s);
  }
  {  // per (X, m): s2[m][X][a,Y] = Aq[(m,a),(A',n)] @ s1[X][(A',n),Y]
    GemmArgs g;
    g.M = Ra; g.N = rY; g.K = RA * n;
    gemm_set_A(g, Aq, (long long)RA * n, false);
    g.a_bs2 = (long long)Ra * RA * n;
    gemm_set_B(g, s1, rY, false);
    g.b_bs1 = (long long)RA * n * rY;
    gemm_set_C(g, s2, rY);
    g.c_bs1 = (long long)Ra * rY;
    g.c_bs2 = (long long)rX * Ra * rY;
    g.batch1 = rX; g.batch2 = m;
    gemm(g, s);
  }
  {  // out[B,(a,Y)] = bra[B,(m,X)] @ s2[(m,X),(a,Y)]
    GemmArgs g;
    g.M = rB; g.N = Ra * rY; g.K = m * rX;
    gemm_set_A(g, bra, (long long)m * rX, false);
    gemm_set_B(g, s2, (long long)Ra * rY, false);
    gemm_set_C(g, out, (long long)Ra * rY);
    gemm(g, s, sc.p, sc.n);
  }
}

// ---------------------------------------------------------------- local matvec
long long local_matvec_scratch(int rX, int Ra, int rU, int m, int n, int Rb, int rY, int rV) {
  return (long long)rX * Ra * n * rV + (long long)rX * m * Rb * rV + (long long)(rU + 1) * n * rV +
         std::max(splitk_ws(rX * Ra, n * rV, rU), splitk_ws(rX * m, rY, Rb * rV));
}

void local_matvec(const double* phil, int rX, int Ra, int rU, const double* Ap, int m, int n, int Rb,
                  const double* phir, int rY, int rV, const double* v, double* y, double alpha,
                  double beta, Scratch sc, cudaStream_t s, const int* skip) {
  double* t1 = take(sc, (long long)rX * Ra * n * rV).p;  // [X][a][n][V]
  double* t2 = take(sc, (long long)rX * m * Rb * rV).p;  // [X][m][b][V]
  {  // t1[(X,a),(n,V)] = phil[(X,a),U] @ v[U,(n,V)]
    GemmArgs g;
    g.M = rX * Ra; g.N = n * rV; g.K = rU;
    gemm_set_A(g, phil, rU, false);
    if (skip == nullptr && step1_transposed(rX, Ra, rU, n, rV)) {
      const long long ldt = rU + (rU & 1);  // 16-byte row pitch for the tensor map
      double* vT = take(sc, ldt * n * rV).p;  // [(n,V)][U]
      transpose_rows(v, vT, rU, (long long)n * rV, ldt, s);
      g.B = vT; g.b_rs = 1; g.b_cs = ldt;
    } else {
      gemm_set_B(g, v, (long long)n * rV, false);
    }
    gemm_set_C(g, t1, (long long)n * rV);
    g.skip = skip;
    gemm(g, s, sc.p, sc.n);
  }
  {  // per X: t2[X][(m,b),V] = Ap[(m,b),(a,n)] @ t1[X][(a,n),V]
    GemmArgs g;
    g.M = m * Rb; g.N = rV; g.K = Ra * n;
    gemm_set_A(g, Ap, (long long)Ra * n, false);
    gemm_set_B(g, t1, rV, false);
    g.b_bs1 = (long long)Ra * n * rV;
    gemm_set_C(g, t2, rV);
    g.c_bs1 = (long long)m * Rb * rV;
    g.batch1 = rX;
    g.skip = skip;
    gemm(g, s);
  }
  {  // y[(X,m),Y] = alpha * t2[(X,m),(b,V)] @ phir[Y,(b,V)]^T + beta * y
    GemmArgs g;
    g.M = rX * m; g.N = rY; g.K = Rb * rV;
    gemm_set_A(g, t2, (long long)Rb * rV, false);
    gemm_set_B(g, phir, (long long)Rb * rV, true);
    gemm_set_C(g, y, rY);
    g.alpha = alpha; g.beta = beta;
    g.skip = skip;
    gemm(g, s, sc.p, sc.n);
  }
}

// ---------------------------------------------------------------- rhs projections
void psi_left(const double* psi, int rX, int rF, const double* bra, int m, int rU, const double* f,
              int rG, double* out, Scratch sc, cudaStream_t s) {
  double* t = take(sc, (long long)rX * m * rG).p;  // [X][m][G]
  GemmArgs g;
  g.M = rX; g.N = m * rG; g.K = rF;
  gemm_set_A(g, psi, rF, false);
  gemm_set_B(g, f, (long long)m * rG, false);
  gemm_set_C(g, t, (long long)m * rG);
  gemm(g, s);
  GemmArgs h;  // out[U,G] = bra[(X,m),U]^T @ t[(X,m),G]
  h.M = rU; h.N = rG; h.K = rX * m;
  gemm_set_A(h, bra, rU, true);
  gemm_set_B(h, t, rG, false);
  gemm_set_C(h, out, rG);
  gemm(h, s, sc.p, sc.n);
}

void psi_right(const double* psi, int rX, int rG, const double* bra, int rU, int m, const double* f,
               int rF, double* out, Scratch sc, cudaStream_t s) {
  double* t = take(sc, (long long)rF * m * rX).p;  // [F][m][X]
  GemmArgs g;  // t[(F,m),X] = f[(F,m),G] @ psi[X,G]^T
  g.M = rF * m; g.N = rX; g.K = rG;
  gemm_set_A(g, f, rG, false);
  gemm_set_B(g, psi, rG, true);
  gemm_set_C(g, t, rX);
  gemm(g, s);
  GemmArgs h;  // out[U,F] = bra[U,(m,X)] @ t[F,(m,X)]^T
  h.M = rU; h.N = rF; h.K = m * rX;
  gemm_set_A(h, bra, (long long)m * rX, false);
  gemm_set_B(h, t, (long long)m * rX, true);
  gemm_set_C(h, out, rF);
  gemm(h, s, sc.p, sc.n);
}

void local_rhs(const double* psil, int rX, int rF, const double* f, int m, int rG, const double* psir,
               int rY, double* out, Scratch sc, cudaStream_t s) {
  double* t = take(sc, (long long)rX * m * rG).p;  // [X][m][G]
  GemmArgs g;
  g.M = rX; g.N = m * rG; g.K = rF;
  gemm_set_A(g, psil, rF, false);
  gemm_set_B(g, f, (long long)m * rG, false);
  gemm_set_C(g, t, (long long)m * rG);
  gemm(g, s);
  GemmArgs h;  // out[(X,m),Y] = t[(X,m),G] @ psir[Y,G]^T
  h.M = rX * m; h.N = rY; h.K = rG;
  gemm_set_A(h, t, rG, false);
  gemm_set_B(h, psir, rG, true);
  gemm_set_C(h, out, rY);
  gemm(h, s, sc.p, sc.n);
}

// ---------------------------------------------------------------- dense local matrix
long long local_dense_scratch(int rX, int Ra, int rU, int m, int n, int Rb) {
  (void)Ra;
  return (long long)rX * m * rU * n * Rb;
}

void local_dense(const double* phil, int rX, int Ra, int rU, const double* A, int m, int n, int Rb,
                 const double* phir, int rY, int rV, double* mat, Scratch sc, cudaStream_t s) {
  const long long dim = (long long)rU * n * rV;  // columns (U,n,V); rows (X,m,Y)
  double* T1 = take(sc, (long long)rX * m * rU * n * Rb).p;  // [X][m][U][n][b]
  {  // per (X, m): T1[X][m][U,(n,b)] = phil[X]^T[U,a] @ A[a, m, (n,b)]
    GemmArgs g;
    g.M = rU; g.N = n * Rb; g.K = Ra;
    g.A = phil; g.a_rs = 1; g.a_cs = rU; g.a_bs1 = (long long)Ra * rU;
    g.B = A; g.b_rs = (long long)m * n * Rb; g.b_cs = 1; g.b_bs2 = (long long)n * Rb;
    g.C = T1; g.c_rs = (long long)n * Rb; g.c_cs = 1;
    g.c_bs1 = (long long)m * rU * n * Rb; g.c_bs2 = (long long)rU * n * Rb;
    g.batch1 = rX; g.batch2 = m;
    gemm(g, s);
  }
  {  // per ((X,m), Y): mat row (X,m,Y) = T1[(X,m)][(U,n),b] @ phir[Y][b,V]
    GemmArgs g;
    g.M = rU * n; g.N = rV; g.K = Rb;
    gemm_set_A(g, T1, Rb, false);
    g.a_bs1 = (long long)rU * n * Rb;
    gemm_set_B(g, phir, rV, false);
    g.b_bs2 = (long long)Rb * rV;
    gemm_set_C(g, mat, rV);
    g.c_bs1 = (long long)rY * dim;
    g.c_bs2 = dim;
    g.batch1 = rX * m; g.batch2 = rY;
    gemm(g, s);
  }
}

void local_diag(const double* phil, int rX, int Ra, const double* A, int m, int Rb, const double* phir,
                int rY, double* out, Scratch sc, cudaStream_t s) {
  const int n = m;
  double* t = take(sc, (long long)rX * m * Rb).p;  // [X][m][b]
  {  // per m: t[X, m, b] = sum_a phil[X,a,X] A[a,m,m,b]
    GemmArgs g;
    g.M = rX; g.N = Rb; g.K = Ra;
    g.A = phil; g.a_rs = (long long)Ra * rX + 1; g.a_cs = rX;
    g.B = A; g.b_rs = (long long)m * n * Rb; g.b_cs = 1; g.b_bs1 = (long long)(n + 1) * Rb;
    g.C = t; g.c_rs = (long long)m * Rb; g.c_cs = 1; g.c_bs1 = Rb;
    g.batch1 = m;
    gemm(g, s);
  }
  {  // out[(X,m),Y] = sum_b t[(X,m),b] phir[Y,b,Y]
    GemmArgs g;
    g.M = rX * m; g.N = rY; g.K = Rb;
    gemm_set_A(g, t, Rb, false);
    g.B = phir; g.b_rs = rY; g.b_cs = (long long)Rb * rY + 1;
    gemm_set_C(g, out, rY);
    gemm(g, s);
  }
}

double local_matvec_flops(int rX, int Ra, int rU, int m, int n, int Rb, int rY, int rV) {
  return 2.0 * rX * Ra * rU * n * rV + 2.0 * rX * m * Rb * Ra * n * rV + 2.0 * rX * m * rY * Rb * rV;
}

double env_flops(int rX, int RA, int rY, int m, int n, int RB, int rU, int rZ) {
  return 2.0 * rX * RA * rY * n * rZ + 2.0 * rX * m * RB * RA * n * rZ + 2.0 * rU * RB * rZ * rX * m;
}

}  // namespace qtt
