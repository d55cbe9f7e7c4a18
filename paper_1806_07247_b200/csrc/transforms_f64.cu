// fp64 mode-3 transforms (the paper's own precision: Matlab double).
// K1: Alg. 1 step 1, Eq. (2), Hermitian half only (Eq. (8)).
// K3: Alg. 1 step 2 second branch + step 3 (L177-179): conjugate fill fused into the inverse, 1/n3.
//
// In-shared-memory mixed-radix Stockham FFT in double precision, O(n3 log n3) per tube: radix-8
// passes while the power-of-two part allows, one radix 4/2 pass for the rest, then radix-3 and
// radix-5 passes, each R-point DFT held in registers (double2).  n3 that is not 5-smooth goes
// through Bluestein's chirp-z transform of a 5-smooth length M >= 2 n3 - 1 when n3 > 64 (the same
// route as the fp32 path, R12), with chirp and filter computed on the host in fp64; smaller
// non-smooth n3 keep the direct O(n3^2) kernels of transforms.cu (measured faster, e.g. n3 = 31).
//
// Two real tubes x, y share one complex FFT z = x + i y:
//   forward:  X_f = (Z_f + conj Z_{N-f}) / 2,  Y_f = (Z_f - conj Z_{N-f}) / (2i),  f = 0..N/2;
//   inverse:  Z_f = X_f + i Y_f with X_{N-f} = conj X_f (Im of DC / Nyquist dropped), z = IFFT(Z),
//             x = Re z / N, y = Im z / N.
// There is no operand scaling in fp64 (no fp16 split), so pairing two tubes of different
// magnitudes costs nothing beyond fp64 rounding of the larger one (~1e-16 relative), far below
// the 1e-12 tolerance of the fp64 path.
//
// A CTA owns TUB = 2F consecutive tubes of one lateral index q, F = the largest power of two with
// F * L <= 8192 complex points (L = N, or M for Bluestein; <= 128 KB of data + padding), F <= 128.
// Spectra leave as fp64 planes [f][re|im][q][ld] (the fp64 GEMM's operand layout).
#include "internal.h"

#include <complex>
#include <map>
#include <math.h>
#include <mutex>
#include <vector>

namespace tprod {

namespace {

constexpr int PTS64 = 8192;        // complex points per CTA
constexpr int NT64 = 512;          // threads per CTA
constexpr int MAXP64 = 24;

struct Plan64 {
  int np;
  int R[MAXP64];
  int Ns[MAXP64];
  int toff[MAXP64];
};

bool make_plan64(int n, Plan64* pl) {
  if (n < 2) return false;
  int m = n, a = 0;
  while (m % 2 == 0) { m /= 2; ++a; }
  int b = 0, c = 0;
  while (m % 3 == 0) { m /= 3; ++b; }
  while (m % 5 == 0) { m /= 5; ++c; }
  if (m != 1) return false;
  std::vector<int> rs;
  while (a >= 3) { rs.push_back(8); a -= 3; }
  if (a > 0) rs.push_back(1 << a);
  for (int i = 0; i < b; ++i) rs.push_back(3);
  for (int i = 0; i < c; ++i) rs.push_back(5);
  if ((int)rs.size() > MAXP64) return false;
  pl->np = (int)rs.size();
  int Ns = 1, off = 0;
  for (int i = 0; i < pl->np; ++i) {
    pl->R[i] = rs[i];
    pl->Ns[i] = Ns;
    pl->toff[i] = off;
    if (Ns > 1) off += (rs[i] - 1) * Ns;
    Ns *= rs[i];
  }
  return true;
}

size_t table_len64(const Plan64& pl) {
  const int last = pl.np - 1;
  return (size_t)pl.toff[last] + (pl.Ns[last] > 1 ? (size_t)(pl.R[last] - 1) * pl.Ns[last] : 0) + 1;
}

// ---- double2 arithmetic
__device__ __forceinline__ double2 dadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 dsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 dmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 dscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 dmul_i(double2 a) { return make_double2(-a.y, a.x); }

// In-register DFT of R in {2, 3, 4, 5, 8} points, natural order in and out; DIR = -1 forward
// (w = e^{-2 pi i / R}), +1 inverse.
template <int R, int DIR>
__device__ __forceinline__ void dft64(double2 (&v)[R]) {
  if constexpr (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = dadd(a, b);
    v[1] = dsub(a, b);
  } else if constexpr (R == 3) {
    const double c = -0.5, s = DIR * 0.86602540378443864676;
    const double2 t1 = dadd(v[1], v[2]), d = dsub(v[1], v[2]);
    const double2 m = make_double2(v[0].x + c * t1.x, v[0].y + c * t1.y);
    const double2 id = dmul_i(dscale(d, s));
    v[0] = dadd(v[0], t1);
    v[1] = dadd(m, id);
    v[2] = dsub(m, id);
  } else if constexpr (R == 4) {
    const double2 a = dadd(v[0], v[2]), b = dsub(v[0], v[2]);
    const double2 c = dadd(v[1], v[3]), d = dsub(v[1], v[3]);
    // w_4^1 = -i (forward), +i (inverse)
    const double2 dw = DIR < 0 ? make_double2(d.y, -d.x) : make_double2(-d.y, d.x);
    v[0] = dadd(a, c);
    v[2] = dsub(a, c);
    v[1] = dadd(b, dw);
    v[3] = dsub(b, dw);
  } else if constexpr (R == 5) {
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double s1 = DIR * 0.95105651629515357212, s2 = DIR * 0.58778525229247312917;
    const double2 a1 = dadd(v[1], v[4]), b1 = dsub(v[1], v[4]);
    const double2 a2 = dadd(v[2], v[3]), b2 = dsub(v[2], v[3]);
    const double2 m1 = make_double2(v[0].x + c1 * a1.x + c2 * a2.x, v[0].y + c1 * a1.y + c2 * a2.y);
    const double2 m2 = make_double2(v[0].x + c2 * a1.x + c1 * a2.x, v[0].y + c2 * a1.y + c1 * a2.y);
    const double2 n1 = dmul_i(make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
    const double2 n2 = dmul_i(make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
    v[0] = dadd(v[0], dadd(a1, a2));
    v[1] = dadd(m1, n1);
    v[4] = dsub(m1, n1);
    v[2] = dadd(m2, n2);
    v[3] = dsub(m2, n2);
  } else {
    static_assert(R == 8, "radix");
    // two radix-4 DFTs of the even / odd points, twiddles w_8^k, radix-2 combine
    double2 e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
    dft64<4, DIR>(e);
    dft64<4, DIR>(o);
    const double r = 0.70710678118654752440;
    // o[k] *= w_8^{k}: w_8^1 = (r, DIR r), w_8^2 = (0, DIR), w_8^3 = (-r, DIR r)
    o[1] = dmul(o[1], make_double2(r, DIR * r));
    o[2] = DIR < 0 ? make_double2(o[2].y, -o[2].x) : make_double2(-o[2].y, o[2].x);
    o[3] = dmul(o[3], make_double2(-r, DIR * r));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = dadd(e[k], o[k]);
      v[k + 4] = dsub(e[k], o[k]);
    }
  }
}

// padded smem index (one double2 per 16) and an odd buffer stride (lanes of different buffers
// start in different 16-byte bank groups)
__host__ __device__ __forceinline__ int pad64(int i) { return i + (i >> 4); }
__host__ __device__ __forceinline__ int bstride64(int n) {
  const int pl = n + n / 16 + 1;
  return pl | 1;
}

template <int DIR>
__device__ __forceinline__ double2 tw64(const double2* __restrict__ t, int m) {
  const double2 w = __ldg(t + m);
  return make_double2(w.x, DIR < 0 ? -w.y : w.y);
}

// One Stockham pass (radix R, span Ns) over the F buffers (stride Np); butterfly b -> buffer
// c = b / NB, j = b mod NB, k = j mod Ns:
//   v[r] = z[j + r NB] w_{Ns R}^{r k};  v = DFT_R(v);  z[(j - k) R + k + r Ns] = v[r].
// In place: every thread loads ALL of its butterflies into registers (F N <= PTS64 points over
// NT64 threads), the CTA synchronises, then writes.
template <int R, int DIR>
__device__ __forceinline__ void pass64(double2* z, int N, int F, int Np, int Ns, const double2* __restrict__ tp) {
  constexpr int BPT = (PTS64 / R + NT64 - 1) / NT64;
  const int NB = N / R;
  const int total = F * NB;
  double2 v[BPT][R];
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    // past-the-end butterflies redo the last one (their results are not stored)
    const int b = min((int)threadIdx.x + u * NT64, total - 1);
    const int c = b / NB, j = b - c * NB, k = j % Ns;
    const double2* zc = z + c * Np;
#pragma unroll
    for (int r = 0; r < R; ++r) v[u][r] = zc[pad64(j + r * NB)];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[u][r] = dmul(v[u][r], tw64<DIR>(tp, (r - 1) * Ns + k));
    }
    dft64<R, DIR>(v[u]);
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < BPT; ++u) {
    const int b = (int)threadIdx.x + u * NT64;
    if (b < total) {
      const int c = b / NB, j = b - c * NB, k = j % Ns;
      double2* zc = z + c * Np;
      const int d0 = (j - k) * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) zc[pad64(d0 + r * Ns)] = v[u][r];
    }
  }
  __syncthreads();
}

// Plan of one transform length: the FFT itself (M = 0) or Bluestein of length N through a
// length-M FFT.
struct Job64 {
  int M;
  const double2* chirp;   // c_k = e^{-pi i k^2 / N}
  const double2* bh;      // FFT_M(b) / M, b_m = conj(c_m) wrapped cyclically
};

template <int DIR>
__device__ void fft64_smem(double2* z, int N, int F, int Np, const Plan64& pl, const double2* __restrict__ st) {
  for (int i = 0; i < pl.np; ++i) {
    const double2* tp = st + pl.toff[i];
    switch (pl.R[i]) {
      case 8: pass64<8, DIR>(z, N, F, Np, pl.Ns[i], tp); break;
      case 4: pass64<4, DIR>(z, N, F, Np, pl.Ns[i], tp); break;
      case 2: pass64<2, DIR>(z, N, F, Np, pl.Ns[i], tp); break;
      case 3: pass64<3, DIR>(z, N, F, Np, pl.Ns[i], tp); break;
      default: pass64<5, DIR>(z, N, F, Np, pl.Ns[i], tp); break;
    }
  }
}

// Bluestein: Z_f = c_f sum_k (z_k c_k) b_{f-k} = c_f IFFT_M(FFT_M(z c) . FFT_M(b)) (bh carries 1/M).
__device__ void bluestein64(double2* z, int N, int M, int F, int Np, const Plan64& pl,
                            const double2* __restrict__ st, const double2* __restrict__ chirp,
                            const double2* __restrict__ bh) {
  for (int idx = threadIdx.x; idx < F * M; idx += NT64) {
    const int c = idx / M, k = idx - c * M;
    double2* e = z + c * Np + pad64(k);
    *e = k < N ? dmul(*e, __ldg(chirp + k)) : make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft64_smem<-1>(z, M, F, Np, pl, st);
  for (int idx = threadIdx.x; idx < F * M; idx += NT64) {
    const int c = idx / M, k = idx - c * M;
    double2* e = z + c * Np + pad64(k);
    *e = dmul(*e, __ldg(bh + k));
  }
  __syncthreads();
  fft64_smem<+1>(z, M, F, Np, pl, st);
  for (int idx = threadIdx.x; idx < F * N; idx += NT64) {
    const int c = idx / N, f = idx - c * N;
    double2* e = z + c * Np + pad64(f);
    *e = dmul(*e, __ldg(chirp + f));
  }
  __syncthreads();
}

template <int DIR>
__device__ void fft64_core(double2* z, int N, int F, int Np, const Plan64& pl, const double2* __restrict__ st,
                           const Job64& job) {
  if (!job.M) {
    fft64_smem<DIR>(z, N, F, Np, pl, st);
    return;
  }
  if (DIR < 0) {
    bluestein64(z, N, job.M, F, Np, pl, st, job.chirp, job.bh);
  } else {                                            // inverse DFT = conj(DFT(conj z))
    for (int idx = threadIdx.x; idx < F * N; idx += NT64) {
      double2* e = z + (idx / N) * Np + pad64(idx % N);
      e->y = -e->y;
    }
    __syncthreads();
    bluestein64(z, N, job.M, F, Np, pl, st, job.chirp, job.bh);
    for (int idx = threadIdx.x; idx < F * N; idx += NT64) {
      double2* e = z + (idx / N) * Np + pad64(idx % N);
      e->y = -e->y;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(NT64, 1) fft64_fwd_kernel(const double* __restrict__ X, int64_t P, int64_t Q, int N,
                                                        int F, const __grid_constant__ Plan64 pl,
                                                        const double2* __restrict__ st, Job64 job,
                                                        double* __restrict__ out, int64_t ld) {
  extern __shared__ double2 z64[];
  const int TUB = 2 * F;
  const int Np = bstride64(job.M ? job.M : N);
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int64_t PQ = P * Q;
  const double* x = X + P * q + p0;
  // tube p0 + t, element k -> buffer t / 2, real (t even) / imaginary (t odd) part
  for (int idx = threadIdx.x; idx < TUB * N; idx += NT64) {
    const int t = idx % TUB, k = idx / TUB;
    const double v = (p0 + t < P) ? __ldg(x + PQ * k + t) : 0.0;
    reinterpret_cast<double*>(z64 + (t >> 1) * Np + pad64(k))[t & 1] = v;
  }
  __syncthreads();
  fft64_core<-1>(z64, N, F, Np, pl, st, job);
  const int H = N / 2 + 1;
  const int64_t plane = Q * ld;
  for (int idx = threadIdx.x; idx < H * F; idx += NT64) {
    const int c = idx % F, f = idx / F;
    const int64_t p = p0 + 2 * c;
    if (p >= P) continue;
    const double2 zf = z64[c * Np + pad64(f)];
    const double2 zm = z64[c * Np + pad64(f == 0 ? 0 : N - f)];
    double* o = out + q * ld + p + (int64_t)(2 * f) * plane;
    o[0] = 0.5 * (zf.x + zm.x);                      // Re X_f
    o[plane] = 0.5 * (zf.y - zm.y);                  // Im X_f
    if (p + 1 < P) {
      o[1] = 0.5 * (zf.y + zm.y);                    // Re Y_f
      o[plane + 1] = -0.5 * (zf.x - zm.x);           // Im Y_f
    }
  }
}

__global__ void __launch_bounds__(NT64, 1) fft64_inv_kernel(const double* __restrict__ Cb, int64_t ld, int64_t P,
                                                        int64_t Q, int N, int F, const __grid_constant__ Plan64 pl,
                                                        const double2* __restrict__ st, Job64 job,
                                                        double* __restrict__ X) {
  extern __shared__ double2 z64[];
  const int TUB = 2 * F;
  const int Np = bstride64(job.M ? job.M : N);
  const int64_t pblocks = (P + TUB - 1) / TUB;
  const int64_t q = blockIdx.x / pblocks;
  const int64_t p0 = (blockIdx.x - q * pblocks) * TUB;
  const int H = N / 2 + 1;
  const int64_t plane = Q * ld;
  for (int idx = threadIdx.x; idx < H * F; idx += NT64) {
    const int c = idx % F, f = idx / F;
    const int64_t p = p0 + 2 * c;
    const double* cr = Cb + (int64_t)(2 * f) * plane + q * ld + p;
    const bool self = (f == 0 || 2 * f == N);        // DC / Nyquist: imaginary part dropped (C2R)
    double xr = 0.0, xi = 0.0, yr = 0.0, yi = 0.0;
    if (p < P) { xr = __ldg(cr); if (!self) xi = __ldg(cr + plane); }
    if (p + 1 < P) { yr = __ldg(cr + 1); if (!self) yi = __ldg(cr + plane + 1); }
    z64[c * Np + pad64(f)] = make_double2(xr - yi, xi + yr);                 // X_f + i Y_f
    if (!self) z64[c * Np + pad64(N - f)] = make_double2(xr + yi, yr - xi);  // conj X_f + i conj Y_f
  }
  __syncthreads();
  fft64_core<+1>(z64, N, F, Np, pl, st, job);
  const int64_t PQ = P * Q;
  const double inv_n = 1.0 / (double)N;
  double* xo = X + P * q + p0;
  for (int idx = threadIdx.x; idx < TUB * N; idx += NT64) {
    const int t = idx % TUB, k = idx / TUB;
    if (p0 + t >= P) continue;
    const double2 v = z64[(t >> 1) * Np + pad64(k)];
    xo[PQ * k + t] = ((t & 1) == 0 ? v.x : v.y) * inv_n;
  }
}

// ---- host tables (cached per device and length; built outside any stream capture by
// fft64_prepare, so the launches themselves never allocate)
struct Tabs64 {
  int N = 0;           // transform length
  int L = 0;           // FFT length actually run (N, or Bluestein's M)
  Plan64 pl{};
  const double2* st = nullptr;
  Job64 job{0, nullptr, nullptr};
};

void host_fft64(std::vector<std::complex<double>>& a) {   // recursive mixed-radix DIT, sign -1
  const int n = (int)a.size();
  if (n == 1) return;
  const int r = n % 2 == 0 ? 2 : n % 3 == 0 ? 3 : 5;
  const int m = n / r;
  std::vector<std::vector<std::complex<double>>> sub(r, std::vector<std::complex<double>>(m));
  for (int j = 0; j < m; ++j)
    for (int q = 0; q < r; ++q) sub[q][j] = a[j * r + q];
  for (int q = 0; q < r; ++q) host_fft64(sub[q]);
  std::vector<double> cs(2 * (size_t)n);
  host_twiddles(n, cs.data());
  for (int k = 0; k < n; ++k) {
    std::complex<double> acc = 0.0;
    for (int q = 0; q < r; ++q) {
      const long long mm = ((long long)q * k) % n;                 // w_n^{qk} = (cos, -sin)
      acc += sub[q][k % m] * std::complex<double>(cs[2 * mm], -cs[2 * mm + 1]);
    }
    a[k] = acc;
  }
}

template <typename T>
const T* upload(const std::vector<T>& v) {
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(T) * v.size()) != cudaSuccess) { cudaGetLastError(); return nullptr; }
  if (cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return (const T*)d;
}

const double2* stockham64(int n, const Plan64& pl) {
  std::vector<double> cs(2 * (size_t)n);
  host_twiddles(n, cs.data());
  std::vector<double2> t(table_len64(pl));
  for (int i = 0; i < pl.np; ++i) {
    const int R = pl.R[i], Ns = pl.Ns[i];
    if (Ns == 1) continue;
    for (int r = 1; r < R; ++r)
      for (int k = 0; k < Ns; ++k) {
        const long long m = (long long)r * k * (n / (Ns * R));   // w_{Ns R}^{r k} = w_n^m
        t[pl.toff[i] + (size_t)(r - 1) * Ns + k] = make_double2(cs[2 * m], cs[2 * m + 1]);
      }
  }
  return upload(t);
}

bool tables64(int n, Tabs64* out) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, Tabs64> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, n});
  if (it != cache.end()) { *out = it->second; return out->L > 0; }
  Tabs64 t;
  t.N = n;
  if (n >= 2 && make_plan64(n, &t.pl)) {
    t.L = n;
    t.st = stockham64(n, t.pl);
    if (!t.st) t.L = 0;
  } else if (n > 64) {              // small non-smooth n3: the direct O(n3^2) kernel is faster
    int M = 0;
    for (int m = 2 * n - 1; m <= PTS64; ++m)
      if (make_plan64(m, &t.pl)) { M = m; break; }
    if (M) {
      std::vector<double2> chirp(n), bh(M);
      std::vector<std::complex<double>> b(M, 0.0);
      std::vector<double> cs2(4 * (size_t)n);
      host_twiddles(2 * n, cs2.data());
      for (int k = 0; k < n; ++k) {
        const long long m = ((long long)k * k) % (2LL * n);
        const double c = cs2[2 * m], s = cs2[2 * m + 1];
        chirp[k] = make_double2(c, -s);
        b[k] = std::complex<double>(c, s);
        if (k) b[M - k] = b[k];
      }
      host_fft64(b);
      for (int k = 0; k < M; ++k) bh[k] = make_double2(b[k].real() / M, b[k].imag() / M);
      t.L = M;
      t.st = stockham64(M, t.pl);
      t.job = Job64{M, upload(chirp), upload(bh)};
      if (!t.st || !t.job.chirp || !t.job.bh) t.L = 0;
    }
  }
  cache[{dev, n}] = t;
  *out = t;
  return t.L > 0;
}

int F_of64(int L) {
  int F = 1;
  while (2 * F * L <= PTS64 && F < 128) F *= 2;
  return F;
}

size_t smem64(int L, int F) { return sizeof(double2) * (size_t)F * bstride64(L); }

}  // namespace

bool fft64_prepare(int64_t n3) {
  if (n3 < 2 || n3 > PTS64) return false;
  Tabs64 t;
  return tables64((int)n3, &t);
}

bool launch_fwd_fft64(const double* X, int64_t P, int64_t Q, int64_t n3, double* out, int64_t ld, cudaStream_t s) {
  if (n3 < 2 || n3 > PTS64) return false;
  Tabs64 t;
  if (!tables64((int)n3, &t)) return false;
  const int F = F_of64(t.L);
  const size_t smem = smem64(t.L, F);
  if (cudaFuncSetAttribute((const void*)fft64_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int64_t blocks = (P + 2 * F - 1) / (2 * F) * Q;
  fft64_fwd_kernel<<<(unsigned)blocks, NT64, smem, s>>>(X, P, Q, (int)n3, F, t.pl, t.st, t.job, out, ld);
  return cudaGetLastError() == cudaSuccess;
}

bool launch_inv_fft64(const double* Cb, int64_t ld, int64_t P, int64_t Q, int64_t n3, double* X, cudaStream_t s) {
  if (n3 < 2 || n3 > PTS64) return false;
  Tabs64 t;
  if (!tables64((int)n3, &t)) return false;
  const int F = F_of64(t.L);
  const size_t smem = smem64(t.L, F);
  if (cudaFuncSetAttribute((const void*)fft64_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  const int64_t blocks = (P + 2 * F - 1) / (2 * F) * Q;
  fft64_inv_kernel<<<(unsigned)blocks, NT64, smem, s>>>(Cb, ld, P, Q, (int)n3, F, t.pl, t.st, t.job, X);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace tprod
