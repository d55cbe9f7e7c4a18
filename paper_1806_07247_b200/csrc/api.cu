// C ABI of libtprod.so (include/tprod.h): handle, validation, plan/tables, workspace and the
// launch sequence of the hot path (Algorithm 1):
//
//   fp32:  K0 absmax(A), K0 absmax(B)            exact power-of-two operand scales
//          K1 fwd_split(A), K1 fwd_split(B)      Alg. 1 step 1 on the Hermitian half
//          K2 gemm (tcgen05; SIMT reference)     Alg. 1 step 2, first branch (h slices)
//          K3 inv                                Alg. 1 step 2 second branch + step 3, fused
//   fp64:  K1 fwd_f64 x2 (mixed-radix / Bluestein fp64 FFT, transforms_f64.cu), K2 gemm_simt_f64, K3 inv_f64
#include "../../include/tprod.h"
#include "internal.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

using namespace tprod;

// Prepared left operand (tprod_prepare_a_f32): A's row unscale vector and split spectrum planes.
struct PreparedA {
  bool valid = false;
  int64_t n1 = 0, n2 = 0, n3 = 0, lda = 0, h = 0;
  void* buf = nullptr;
  size_t bytes = 0;
  unsigned* maxA = nullptr;
  float* uA = nullptr;
  __half* Ab = nullptr;
};

struct tprod_ctx {
  int device = 0;
  int num_sms = 148;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  std::map<int, float2*> tw32;
  std::map<int, float2*> st32;   // Stockham FFT tables (power-of-two n3 > 64)
  std::map<int, double2*> tw64;
  void* hbuf[3] = {nullptr, nullptr, nullptr};   // device buffers of the *_host entry points
  size_t hbuf_bytes[3] = {0, 0, 0};
  int64_t last_launches = 0;
  int engine = 0;
  int force_bn = 0;
  int force_cn = 0;
  int transform = 0;   // TPROD_OPT_TRANSFORM
  void* comm = nullptr;  // ncclComm_t
  int rank = 0, world = 1;
  bool timing = false;
  bool timed_last = false;
  bool forked_last = false;           // the last timed call ran the A / B chains concurrently
  bool overlap = true;                // TPROD_OPT_OVERLAP: K3 as a programmatic dependent of the GEMM
  bool overlap_stream = true;         // ... also for many-round GEMMs with the streaming tube inverse (off with value 2)
  bool fused_scales = true;           // TPROD_OPT_FUSED_SCALES: K0 of B inside K1 of B (n3 <= 32)
  bool overlapped_last = false;       // the last timed call overlapped K2 and K3 (one stage)
  int* done = nullptr;                // OVERLAP_COUNTERS (m, n) tile counters (internal.h OverlapK3)
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  PreparedA prep;
  // pipelined host entry point (tprod_f32_host): copy streams, double-buffer events, its own A
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  PreparedA prep_host;
  // CUDA-graph cache of the launch sequence (TPROD_OPT_GRAPHS): key = everything the kernels'
  // parameters derive from (operand / workspace / table pointers, shapes, options)
  bool graphs = true;
  bool poison = false;                                 // TPROD_OPT_POISON: NaN-fill the workspace before each call
  bool sync_checks = true;                             // TPROD_OPT_SYNC_CHECKS
  int* status = nullptr;                               // device status word (TPROD_STATUS_* bits), tprod_status
  cudaStream_t cap = nullptr;                          // private capture stream
  // small problems: K1 of A on a side stream concurrently with K1 of B (fork / join by events)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    int seen = 0;                                      // direct runs before capture (< 0: capture failed, never retry)
    int64_t launches = 0;
  };
  std::map<std::vector<int64_t>, GraphEntry> graph_cache;
  // buffers from cudaMallocAsync (released with cudaFreeAsync); buffers replaced while a stream was
  // being captured are kept in `retired` until tprod_destroy
  std::map<void*, bool> async_buf;
  std::vector<void*> retired;
};

namespace {

#define CK(call)                                   \
  do {                                             \
    cudaError_t _e = (call);                       \
    if (_e != cudaSuccess) {                       \
      return TPROD_ECUDA;                          \
    }                                              \
  } while (0)

bool checked_mul(int64_t a, int64_t b, int64_t* out) {
  if (a < 0 || b < 0) return false;
  if (a != 0 && b > INT64_MAX / a) return false;
  *out = a * b;
  return true;
}

int validate_dims(int64_t n1, int64_t n2, int64_t n3, int64_t n4) {
  if (n1 < 1 || n2 < 1 || n3 < 1 || n4 < 1) return TPROD_EINVAL;
  const int64_t lim = (int64_t)1 << 31;
  if (n1 >= lim || n2 >= lim || n3 >= lim || n4 >= lim) return TPROD_EINVAL;
  int64_t t;
  if (!checked_mul(n1, n2, &t) || !checked_mul(t, n3, &t) || t > ((int64_t)1 << 40)) return TPROD_EINVAL;
  if (!checked_mul(n2, n4, &t) || !checked_mul(t, n3, &t) || t > ((int64_t)1 << 40)) return TPROD_EINVAL;
  if (!checked_mul(n1, n4, &t) || !checked_mul(t, n3, &t) || t > ((int64_t)1 << 40)) return TPROD_EINVAL;
  if (h_slices(n3) > 65535) return TPROD_EUNSUPPORTED;   // grid.z of the SIMT engines
  if ((n1 + 127) / 128 * n2 >= lim || (n2 + 127) / 128 * n4 >= lim) return TPROD_EUNSUPPORTED;
  return TPROD_OK;
}

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  uintptr_t a0 = (uintptr_t)a, b0 = (uintptr_t)b;
  return a0 < b0 + bn && b0 < a0 + an;
}

// ---------------------------------------------------------------- workspace layout
struct Layout32 {
  int64_t h, lda, ldb, ldc;
  size_t off_maxA, off_maxB, off_uA, off_uB, off_Ab, off_Bb, off_Cb, off_W, W_bytes, off_W2, W2_bytes, total;
};
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Small operands: K1 of A runs on a side stream concurrently with K1 of B (launch_f32).
#ifndef TPROD_FORK_MELEMS
#define TPROD_FORK_MELEMS 256
#endif
#ifndef TPROD_FORK_K0
#define TPROD_FORK_K0 1
#endif
bool fork_dims(int64_t n1, int64_t n2, int64_t n3, int64_t n4) {
  return (n1 * n2 + n2 * n4) * n3 <= (int64_t)TPROD_FORK_MELEMS << 20;
}

// with_A = false: no A-bar region (prepared-operand calls read the handle's prepared planes)
Layout32 layout32(int64_t n1, int64_t n2, int64_t n3, int64_t n4, bool with_A = true) {
  Layout32 L;
  L.h = h_slices(n3);
  L.lda = round_up(n1, 8);   // 16-byte row pitch for TMA (fp16)
  L.ldb = round_up(n2, 8);
  L.ldc = round_up(n1, 4);
  size_t o = 0;
  L.off_maxA = o; o = align_up(o + 4 * (size_t)n1, 1024);
  L.off_maxB = o; o = align_up(o + 4 * (size_t)n4, 1024);
  L.off_uA = o;   o = align_up(o + 4 * (size_t)n1, 1024);
  L.off_uB = o;   o = align_up(o + 4 * (size_t)n4, 1024);
  L.off_Ab = o;  if (with_A) o = align_up(o + 2 * (size_t)(L.h * NPLANES * n2 * L.lda), 1024);
  L.off_Bb = o;   o = align_up(o + 2 * (size_t)(L.h * NPLANES * n4 * L.ldb), 1024);
  L.off_Cb = o;   o = align_up(o + 4 * (size_t)(L.h * 2 * n4 * L.ldc), 1024);
  // four-step long-tube transforms: intermediate the size of the largest tensor they transform
  // (A and B forward, C inverse -- without C's size a prepared-operand call with n1 > n2 fell back
  // to the mixed-radix inverse and differed from the one-shot call in the last bits)
  int f1 = 0, f2 = 0;
  fourstep_factors(n3, &f1, &f2);
  L.W_bytes = f1 ? 4 * (size_t)(std::max({with_A ? n1 * n2 : (int64_t)0, n2 * n4, n1 * n4}) * n3) : 0;
  L.off_W = o;    o = align_up(o + L.W_bytes, 1024);
  // A's own four-step intermediate when K1 of A runs concurrently with K1 of B
  L.W2_bytes = f1 && with_A && fork_dims(n1, n2, n3, n4) ? 4 * (size_t)(n1 * n2 * n3) : 0;
  L.off_W2 = o;   o = align_up(o + L.W2_bytes, 1024);
  L.total = o;
  return L;
}

struct Layout64 {
  int64_t h;
  size_t off_Ab, off_Bb, off_Cb, total;
};
Layout64 layout64(int64_t n1, int64_t n2, int64_t n3, int64_t n4) {
  Layout64 L;
  L.h = h_slices(n3);
  size_t o = 0;
  L.off_Ab = o; o = align_up(o + 8 * (size_t)(L.h * 2 * n1 * n2), 1024);
  L.off_Bb = o; o = align_up(o + 8 * (size_t)(L.h * 2 * n2 * n4), 1024);
  L.off_Cb = o; o = align_up(o + 8 * (size_t)(L.h * 2 * n1 * n4), 1024);
  L.total = o;
  return L;
}

void clear_graphs(tprod_ctx* h);

// Stream-ordered device buffers of the handle (workspace, host-path buffers, prepared operands):
// allocated with cudaMallocAsync on the call's stream and released with cudaFreeAsync on the stream
// of the call that outgrows them, so growing a buffer never synchronises the device (work already
// enqueued on that stream finishes with the old buffer first; a handle is used from one stream at a
// time, include/tprod.h).  While the stream is being captured into a graph, plain cudaMalloc is
// used and an outgrown buffer is kept until tprod_destroy.
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) { cudaGetLastError(); return true; }
  return cs != cudaStreamCaptureStatusNone;
}
int dev_alloc(tprod_ctx* h, void** p, size_t bytes, cudaStream_t s) {
  *p = nullptr;
  if (!capturing(s) && cudaMallocAsync(p, bytes, s) == cudaSuccess) {
    h->async_buf[*p] = true;
    return TPROD_OK;
  }
  cudaGetLastError();
  if (cudaMalloc(p, bytes) != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return TPROD_ENOMEM;
  }
  h->async_buf[*p] = false;
  return TPROD_OK;
}
void dev_release(tprod_ctx* h, void* p, cudaStream_t s) {
  if (!p) return;
  auto it = h->async_buf.find(p);
  const bool async = it != h->async_buf.end() && it->second;
  if (async && !capturing(s) && cudaFreeAsync(p, s) == cudaSuccess) {
    h->async_buf.erase(it);
    return;
  }
  cudaGetLastError();
  h->retired.push_back(p);
}

// Grow-only workspace; the cached graphs address the old buffer and are dropped (an executable
// graph still in flight is released by the driver when it completes).
int ensure_ws(tprod_ctx* h, size_t bytes, cudaStream_t s) {
  if (h->ws_bytes >= bytes) return TPROD_OK;
  if (h->ws) {
    clear_graphs(h);
    dev_release(h, h->ws, s);
    h->ws = nullptr;
    h->ws_bytes = 0;
  }
  int st = dev_alloc(h, &h->ws, bytes, s);
  if (st) return st;
  h->ws_bytes = bytes;
  return TPROD_OK;
}

// TPROD_OPT_POISON: fill `bytes` of the workspace with 0xFF (a NaN pattern in fp32 / fp64 / fp16)
// on the call's stream, so that a kernel reading workspace it did not write first shows up as NaN
// in the result (the stand-in for initcheck, which is not available on the GPU pool).
int poison_ws(tprod_ctx* h, size_t bytes, cudaStream_t s) {
  if (!h->poison || !bytes) return TPROD_OK;
  CK(cudaMemsetAsync(h->ws, 0xFF, std::min(bytes, h->ws_bytes), s));
  return TPROD_OK;
}

int ensure_hbuf(tprod_ctx* h, int which, size_t bytes, cudaStream_t s) {
  if (h->hbuf_bytes[which] >= bytes) return TPROD_OK;
  if (h->hbuf[which]) {
    dev_release(h, h->hbuf[which], s);
    h->hbuf[which] = nullptr;
    h->hbuf_bytes[which] = 0;
  }
  if (int st = dev_alloc(h, &h->hbuf[which], bytes, s)) return st;
  h->hbuf_bytes[which] = bytes;
  return TPROD_OK;
}

int get_tw32(tprod_ctx* h, int n3, const float2** out) {
  auto it = h->tw32.find(n3);
  if (it != h->tw32.end()) { *out = it->second; return TPROD_OK; }
  std::vector<double> cs(2 * (size_t)n3);
  host_twiddles(n3, cs.data());
  std::vector<float2> t(n3);
  for (int m = 0; m < n3; ++m) t[m] = make_float2((float)cs[2 * m], (float)cs[2 * m + 1]);  // RN
  float2* d = nullptr;
  if (cudaMalloc(&d, sizeof(float2) * n3) != cudaSuccess) { cudaGetLastError(); return TPROD_ENOMEM; }
  CK(cudaMemcpy(d, t.data(), sizeof(float2) * n3, cudaMemcpyHostToDevice));
  h->tw32[n3] = d;
  *out = d;
  return TPROD_OK;
}

// The fp32 twiddles of a call: the (cos, sin) table, plus the Stockham FFT table when n3 takes the
// FFT path.
int get_twiddles32(tprod_ctx* h, int n3, Twiddles32* T) {
  const float2* tw = nullptr;
  int st = get_tw32(h, n3, &tw);
  if (st) return st;
  *T = Twiddles32{tw, n3, nullptr};
  int f1 = 0, f2 = 0;
  fourstep_factors(n3, &f1, &f2);
  if (f1) {
    Twiddles32 T1, T2;
    if ((st = get_twiddles32(h, f1, &T1)) || (st = get_twiddles32(h, f2, &T2))) return st;
    T->st_n1 = T1.st;
    T->st_n2 = T2.st;
  }
  if (!fft_supported(n3) && !tube_supported(n3)) return TPROD_OK;
  auto it = h->st32.find(n3);
  if (it != h->st32.end()) { T->st = it->second; return TPROD_OK; }
  std::vector<double> cs(2 * (size_t)n3);
  host_twiddles(n3, cs.data());
  std::vector<float2> t(stockham_table_len(n3) + 1);
  host_stockham_table(n3, cs.data(), t.data());
  float2* d = nullptr;
  if (cudaMalloc(&d, sizeof(float2) * t.size()) != cudaSuccess) { cudaGetLastError(); return TPROD_ENOMEM; }
  CK(cudaMemcpy(d, t.data(), sizeof(float2) * t.size(), cudaMemcpyHostToDevice));
  h->st32[n3] = d;
  T->st = d;
  return TPROD_OK;
}

int get_tw64(tprod_ctx* h, int n3, const double2** out) {
  auto it = h->tw64.find(n3);
  if (it != h->tw64.end()) { *out = it->second; return TPROD_OK; }
  std::vector<double> cs(2 * (size_t)n3);
  host_twiddles(n3, cs.data());
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(double2) * n3) != cudaSuccess) { cudaGetLastError(); return TPROD_ENOMEM; }
  CK(cudaMemcpy(d, cs.data(), sizeof(double2) * n3, cudaMemcpyHostToDevice));
  h->tw64[n3] = d;
  *out = d;
  return TPROD_OK;
}

int launch_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TPROD_OK : TPROD_ECUDA;
}

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // Prefer the NCCL torch already loaded (matched by soname), else the system one.
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(lib, "ncclCommInitRank");
    api.Broadcast = (decltype(api.Broadcast))dlsym(lib, "ncclBroadcast");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(lib, "ncclCommDestroy");
    api.ok = api.GetUniqueId && api.CommInitRank && api.Broadcast && api.CommDestroy;
  });
  return api;
}

// K0 + K1 of A into a PreparedA (tprod_prepare_a_f32 and the pipelined host entry point).  The
// four-step transforms get their intermediate from the handle workspace (stream-ordered with every
// other call on the handle).
int prepare_into(tprod_ctx* h, PreparedA& P, const float* A, int64_t n1, int64_t n2, int64_t n3, cudaStream_t s) {
  int st;
  const int64_t hh = h_slices(n3), lda = round_up(n1, 8);
  const size_t off_u = align_up(4 * (size_t)n1, 1024);
  const size_t off_Ab = off_u + align_up(4 * (size_t)n1, 1024);
  const size_t bytes = off_Ab + 2 * (size_t)(hh * NPLANES * n2 * lda);
  if (P.bytes < bytes) {
    if (P.buf) {
      dev_release(h, P.buf, s);
      P.buf = nullptr;
      P.bytes = 0;
    }
    if ((st = dev_alloc(h, &P.buf, bytes, s))) { P.valid = false; return st; }
    P.bytes = bytes;
  }
  Twiddles32 T;
  if ((st = get_twiddles32(h, (int)n3, &T))) return st;
  T.staged = h->transform != 1;
  T.cluster = h->transform == 3;
  T.tc = h->transform == 2;
  int f1 = 0, f2 = 0;
  fourstep_factors(n3, &f1, &f2);
  if (f1) {
    const size_t w = 4 * (size_t)(n1 * n2 * n3);
    if ((st = ensure_ws(h, w, s))) return st;
    T.scratch = (float*)h->ws;
    T.scratch_bytes = w;
  }
  if (h->poison) CK(cudaMemsetAsync(P.buf, 0xFF, bytes, s));
  if ((st = poison_ws(h, T.scratch_bytes, s))) return st;
  P.maxA = (unsigned*)P.buf;
  P.uA = (float*)((char*)P.buf + off_u);
  P.Ab = (__half*)((char*)P.buf + off_Ab);
  CK(cudaMemsetAsync(P.maxA, 0, 4 * (size_t)n1, s));
  launch_absmax2(A, nullptr, n1, n2, n3, 1, P.maxA, nullptr, h->num_sms, s);               // K0 (A)
  launch_fwd_split(A, n1, n2, n3, 0, P.maxA, T, P.Ab, lda, P.uA, h->num_sms, s);         // K1 (A)
  if ((st = launch_status())) { P.valid = false; return st; }
  P.valid = true;
  P.n1 = n1; P.n2 = n2; P.n3 = n3; P.lda = lda; P.h = hh;
  return TPROD_OK;
}

// ---------------------------------------------------------------- CUDA-graph replay
constexpr size_t GRAPH_CACHE_MAX = 64;

void clear_graphs(tprod_ctx* h) {
  for (auto& kv : h->graph_cache)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  h->graph_cache.clear();
}

// Runs `body(stream)` -- the whole launch sequence of one call, host-side setup (workspace, tables)
// already done -- directly the first time a key is seen and, from the second time on, as one
// cudaGraphLaunch of its captured graph: the per-kernel host work (argument and tensor-map
// encoding, launch calls) of a call with a repeated key is paid once, and the kernels start
// back to back on the device.  A key fixes every kernel parameter, so replay is exactly the direct
// launch sequence on the current contents of the buffers.  Not used while TPROD_OPT_TIMING is on
// (the stage events are recorded between direct launches) or when the caller's stream is itself
// being captured (the launches then join the caller's graph).
template <class Body>
int graph_run(tprod_ctx* h, std::vector<int64_t>&& key, cudaStream_t s, Body&& body) {
  if (!h->graphs || h->timing) return body(s);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone) return body(s);
  auto it = h->graph_cache.find(key);
  if (it == h->graph_cache.end()) {
    if (h->graph_cache.size() >= GRAPH_CACHE_MAX)     // rare: drop the lot (in-flight execs are
      clear_graphs(h);                                 // released by the driver on completion)
    it = h->graph_cache.emplace(std::move(key), tprod_ctx::GraphEntry{}).first;
  }
  tprod_ctx::GraphEntry& e = it->second;
  if (!e.exec) {
    if (e.seen < 1) {                                  // first sighting (or capture failed before): direct
      if (e.seen >= 0) ++e.seen;
      return body(s);
    }
    if (!h->cap) CK(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
    CK(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeRelaxed));
    const int st = body(h->cap);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(h->cap, &g);
    cudaError_t ie = cudaErrorUnknown;
    if (!st && ce == cudaSuccess && g) ie = cudaGraphInstantiate(&e.exec, g, 0);
    if (g) cudaGraphDestroy(g);
    if (ie != cudaSuccess) {                           // not capturable: stay on direct launches
      cudaGetLastError();
      e.exec = nullptr;
      e.seen = -1;
      return body(s);
    }
    e.launches = h->last_launches;
  }
  CK(cudaGraphLaunch(e.exec, s));
  h->last_launches = e.launches;
  h->timed_last = false;
  return TPROD_OK;
}

// ---------------------------------------------------------------- the hot path
// pa != nullptr: A is the handle's prepared operand (A itself is not read; K0/K1 run for B only)
int launch_f32(tprod_ctx* h, const float* A, const float* B, float* C, int64_t n1, int64_t n2, int64_t n3,
               int64_t n4, cudaStream_t s, const PreparedA* pa, const Layout32& L, Twiddles32 T);

int run_f32(tprod_ctx* h, const float* A, const float* B, float* C, int64_t n1, int64_t n2,
            int64_t n3, int64_t n4, cudaStream_t s, const PreparedA* pa = nullptr) {
  Layout32 L = layout32(n1, n2, n3, n4, pa == nullptr);
  int st = ensure_ws(h, L.total, s);
  if (st) return st;
  Twiddles32 T;
  if ((st = get_twiddles32(h, (int)n3, &T))) return st;
  std::vector<int64_t> key = {1, (int64_t)(uintptr_t)A, (int64_t)(uintptr_t)B, (int64_t)(uintptr_t)C, n1, n2, n3, n4,
                              (int64_t)(uintptr_t)h->ws, pa ? (int64_t)(uintptr_t)pa->Ab : 0,
                              pa ? (int64_t)(uintptr_t)pa->uA : 0, pa ? pa->lda : 0, h->engine, h->force_bn,
                              h->force_cn, h->transform, (h->overlap ? 1 : 0) + (h->overlap_stream ? 2 : 0), h->fused_scales ? 1 : 0};
  return graph_run(h, std::move(key), s,
                   [&](cudaStream_t ls) { return launch_f32(h, A, B, C, n1, n2, n3, n4, ls, pa, L, T); });
}

// Side stream + fork / join events of the handle (created with the handle; false = run sequentially).
bool fork_ready(tprod_ctx* h) {
  if (!h->aux && cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    h->aux = nullptr;
    return false;
  }
  if (!h->ev_fork && cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (!h->ev_join && cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

int launch_f32(tprod_ctx* h, const float* A, const float* B, float* C, int64_t n1, int64_t n2, int64_t n3,
               int64_t n4, cudaStream_t s, const PreparedA* pa, const Layout32& L, Twiddles32 T) {
  int st = 0;
  T.staged = h->transform != 1;
  T.cluster = h->transform == 3;
  T.tc = h->transform == 2;
  char* ws = (char*)h->ws;
  T.scratch = L.W_bytes ? (float*)(ws + L.off_W) : nullptr;
  T.scratch_bytes = L.W_bytes;
  unsigned* maxA = (unsigned*)(ws + L.off_maxA);
  unsigned* maxB = (unsigned*)(ws + L.off_maxB);
  float* uA = pa ? pa->uA : (float*)(ws + L.off_uA);
  float* uB = (float*)(ws + L.off_uB);
  __half* Ab = pa ? pa->Ab : (__half*)(ws + L.off_Ab);
  __half* Bb = (__half*)(ws + L.off_Bb);
  float* Cb = (float*)(ws + L.off_Cb);
  int64_t launches = 0;

  auto mark = [&](int i) { if (h->timing) cudaEventRecord(h->ev[i], s); };
  h->timed_last = false;
  if ((st = poison_ws(h, L.total, s))) return st;
  mark(0);
  CK(cudaMemsetAsync(ws + L.off_maxA, 0, L.off_uA - L.off_maxA, s));
  const float* A0 = pa ? nullptr : A;
  // Operands up to TPROD_FORK_MELEMS: the A chain (K0 + K1 of A) runs on a side stream concurrently
  // with the B chain (measured on configs 2, 3 and 4), each K1 right after its own K0
  // (its operand partly still in L2).  Otherwise one K0 launch for both, then B first: the tail of
  // B just streamed by K0 is still resident in L2.
  const bool fork = !pa && fork_dims(n1, n2, n3, n4) && (!L.W_bytes || L.W2_bytes) && fork_ready(h);
  h->forked_last = fork;              // tprod_last_stage_ms: stage 0 = K0 + K1 of both chains, stage 1 = 0
  // K0 of B fused into K1 of B (column scales reduced per lateral slice by a CTA cluster inside the
  // tube-pair transform, n3 <= 32): B is read once instead of twice.  Small B only: measured
  // config 2 (2M elements) 58.1 -> 57.2 us, config 3 (16M, next to the concurrent A chain) 276 -> 284
  // us
  const bool bfused = h->fused_scales && !T.tc && n2 * n4 * n3 <= ((int64_t)8 << 20) && fwd_colmax_ok(B, n2, n3);
  auto k1_B = [&]() -> int {
    if (bfused) return launch_fwd_dense_colmax(B, n2, n4, n3, Bb, L.ldb, uB, s) ? 0 : TPROD_ECUDA;
    launch_fwd_split(B, n2, n4, n3, 1, maxB, T, Bb, L.ldb, uB, h->num_sms, s);   // Alg.1 step 1 (B)
    return 0;
  };
  const float* B0 = bfused ? nullptr : B;       // B's part of K0
  if (fork) {
    Twiddles32 TA = T;                                  // four-step: A's own intermediate
    if (L.W2_bytes) {
      TA.scratch = (float*)(ws + L.off_W2);
      TA.scratch_bytes = L.W2_bytes;
    }
    if (TPROD_FORK_K0) {                                // fork before K0: one K0 launch per chain
      CK(cudaEventRecord(h->ev_fork, s));
      CK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
      launch_absmax2(A, nullptr, n1, n2, n3, 1, maxA, nullptr, h->num_sms, h->aux); ++launches;
      if (B0) {
        launch_absmax2(nullptr, B0, n1, n2, n3, n4, nullptr, maxB, h->num_sms, s);
        ++launches;
      }
    } else {                                            // fork after the shared K0 launch
      launch_absmax2(A0, B0, n1, n2, n3, n4, maxA, maxB, h->num_sms, s);
      launches += (n1 % 4 == 0 && ((uintptr_t)A0 & 15) == 0 && n2 % 4 == 0 && (!B0 || ((uintptr_t)B0 & 15) == 0))
                      ? 1 : (B0 ? 2 : 1);
      CK(cudaEventRecord(h->ev_fork, s));
      CK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
    }
    launch_fwd_split(A, n1, n2, n3, 0, maxA, TA, Ab, L.lda, uA, h->num_sms, h->aux); ++launches;   // Alg.1 step 1 (A)
    CK(cudaEventRecord(h->ev_join, h->aux));
    if ((st = k1_B())) return st;
    ++launches;
    CK(cudaStreamWaitEvent(s, h->ev_join, 0));
  } else {
    if (A0 || B0) {
      launch_absmax2(A0, B0, n1, n2, n3, n4, maxA, maxB, h->num_sms, s);   // row scales of A, col scales of B
      const bool vec = (!A0 || (n1 % 4 == 0 && ((uintptr_t)A0 & 15) == 0)) && n2 % 4 == 0 &&
                       (!B0 || ((uintptr_t)B0 & 15) == 0);
      launches += vec ? 1 : ((A0 ? 1 : 0) + (B0 ? 1 : 0));
    }
    mark(1);
    if ((st = k1_B())) return st;
    ++launches;
    if (!pa) {
      launch_fwd_split(A, n1, n2, n3, 0, maxA, T, Ab, L.lda, uA, h->num_sms, s); ++launches;   // Alg.1 step 1 (A)
    }
  }
  mark(2);
  if ((st = launch_status())) return st;
  bool tc = h->engine == 0 && gemm_tc_supported();
  OverlapK3 ov;
  if (tc) {
    // the counters only where K3 is the tube-pair register kernel (the one that waits on them)
    // ... or the streaming tube inverse of n3 = 64 (any number of tile rounds: config 5)
    ov.stream = h->overlap_stream && T.staged && !T.tc && inv_tube_stream_ok(n1, n3, L.ldc, C);
    int* done = h->overlap && h->done && !T.tc && (inv_dense_pair_ok(n3) || ov.stream) ? h->done : nullptr;
    st = launch_gemm_tc_split(Ab, L.lda, Bb, L.ldb, Cb, L.ldc, n1, n2, n4, L.h, n3 % 2 == 0 ? 1 : 0,
                              h->force_bn, h->force_cn, h->num_sms, s, done, &ov);
    if (st) return st;
  } else {
    launch_gemm_simt_split(Ab, L.lda, Bb, L.ldb, Cb, L.ldc, n1, n2, n4, L.h, s);
  }
  ++launches;                                                     // Alg.1 step 2
  // K3 overlapped with the GEMM's last tile round (internal.h OverlapK3): no event between the two
  // launches (it would serialise them), the stage timer reports K2 + K3 as one stage
  h->overlapped_last = ov.done != nullptr;
  if (!ov.done) mark(3);
  // Alg.1 step 2b + 3; each output tube (i, j) unscaled by uA[i] uB[j] after the inverse (R18)
  launch_inv_f32(Cb, Cb + n4 * L.ldc, L.ldc, 2 * n4 * L.ldc, n1, n4, n3, T, OutUnscale{uA, uB}, C, h->num_sms, s,
                 ov.done ? &ov : nullptr);
  ++launches;
  if (ov.done) mark(3);
  mark(4);
  h->timed_last = h->timing;
  h->last_launches = launches;
  return launch_status();
}

int run_f64(tprod_ctx* h, const double* A, const double* B, double* C, int64_t n1, int64_t n2,
            int64_t n3, int64_t n4, cudaStream_t s) {
  Layout64 L = layout64(n1, n2, n3, n4);
  int st = ensure_ws(h, L.total, s);
  if (st) return st;
  const double2* tw = nullptr;
  if ((st = get_tw64(h, (int)n3, &tw))) return st;
  fft64_prepare(n3);                  // FFT tables built outside any capture (false: generic kernels)
  char* ws = (char*)h->ws;
  double* Ab = (double*)(ws + L.off_Ab);
  double* Bb = (double*)(ws + L.off_Bb);
  double* Cb = (double*)(ws + L.off_Cb);
  Twiddles64 T{tw, (int)n3};
  std::vector<int64_t> key = {2, (int64_t)(uintptr_t)A, (int64_t)(uintptr_t)B, (int64_t)(uintptr_t)C, n1, n2, n3, n4,
                              (int64_t)(uintptr_t)h->ws};
  return graph_run(h, std::move(key), s, [&](cudaStream_t ls) {
    if (int ps = poison_ws(h, L.total, ls)) return ps;
    launch_fwd_f64(A, n1, n2, n3, T, Ab, n1, ls);
    launch_fwd_f64(B, n2, n4, n3, T, Bb, n2, ls);
    launch_gemm_simt_f64(Ab, n1, Bb, n2, Cb, n1, n1, n2, n4, L.h, ls);
    launch_inv_f64(Cb, n1, n1, n4, n3, T, C, ls);
    h->last_launches = 4;
    return launch_status();
  });
}

template <typename T>
int check_call(tprod_ctx* h, const T* A, const T* B, T* C, int64_t n1, int64_t n2, int64_t n3,
               int64_t n4) {
  if (!h || !A || !B || !C) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, n4);
  if (st) return st;
  size_t es = sizeof(T);
  size_t bc = es * (size_t)(n1 * n4 * n3);
  if (overlaps(C, bc, A, es * (size_t)(n1 * n2 * n3)) || overlaps(C, bc, B, es * (size_t)(n2 * n4 * n3)))
    return TPROD_EALIAS;
  return TPROD_OK;
}

// fp32 host entry point, pipelined over lateral-slice chunks (columns of unfold(B) map 1:1 to
// columns of unfold(C), Eq. (9)): A is copied and prepared (K0 + K1 of A) once, then chunk i of B
// is copied in on cs_in while chunk i-1 is computed on `s` (the prepared-operand path) and chunk
// i-2 of C is copied out on cs_out; B / C device chunks are double-buffered.  Every column's result
// is bitwise identical to the one-shot call (prepared path and W-invariance).  Host buffers should
// be pinned for the copies to overlap.
int host_call_f32_pipelined(const float* A, const float* B, float* C, int64_t n1, int64_t n2, int64_t n3,
                            int64_t n4, cudaStream_t s, tprod_handle h, int64_t w) {
  int st;
  if (!h->cs_in) {
    CK(cudaStreamCreateWithFlags(&h->cs_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&h->cs_out, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&h->ev_in[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_comp[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->ev_out[i], cudaEventDisableTiming));
    }
  }
  const size_t bA = 4 * (size_t)(n1 * n2 * n3), bBc = 4 * (size_t)(n2 * w * n3), bCc = 4 * (size_t)(n1 * w * n3);
  if ((st = ensure_hbuf(h, 0, bA, s)) || (st = ensure_hbuf(h, 1, 2 * bBc, s)) || (st = ensure_hbuf(h, 2, 2 * bCc, s))) return st;
  float* dA = (float*)h->hbuf[0];
  float* dB[2] = {(float*)h->hbuf[1], (float*)((char*)h->hbuf[1] + bBc)};
  float* dC[2] = {(float*)h->hbuf[2], (float*)((char*)h->hbuf[2] + bCc)};
  CK(cudaMemcpyAsync(dA, A, bA, cudaMemcpyHostToDevice, s));
  // the copy streams start after everything already on s up to A's copy (earlier work, earlier
  // calls), so B's first chunk streams in while A is prepared
  CK(cudaEventRecord(h->ev_comp[0], s));
  CK(cudaStreamWaitEvent(h->cs_in, h->ev_comp[0], 0));
  CK(cudaStreamWaitEvent(h->cs_out, h->ev_comp[0], 0));
  if ((st = prepare_into(h, h->prep_host, dA, n1, n2, n3, s))) return st;
  const int64_t nch = (n4 + w - 1) / w;
  for (int64_t i = 0; i < nch; ++i) {
    const int b = (int)(i & 1);
    const int64_t j0 = i * w, wi = std::min(w, n4 - j0);
    if (i >= 2) CK(cudaStreamWaitEvent(h->cs_in, h->ev_comp[b], 0));     // compute i-2 has read dB[b]
    // B(:, j0:j0+wi, :): n3 rows of n2*wi floats, host pitch n2*n4
    CK(cudaMemcpy2DAsync(dB[b], 4 * (size_t)(n2 * wi), B + n2 * j0, 4 * (size_t)(n2 * n4), 4 * (size_t)(n2 * wi),
                         (size_t)n3, cudaMemcpyHostToDevice, h->cs_in));
    CK(cudaEventRecord(h->ev_in[b], h->cs_in));
    CK(cudaStreamWaitEvent(s, h->ev_in[b], 0));
    if (i >= 2) CK(cudaStreamWaitEvent(s, h->ev_out[b], 0));            // C chunk i-2 has left dC[b]
    if ((st = run_f32(h, nullptr, dB[b], dC[b], n1, n2, n3, wi, s, &h->prep_host))) return st;
    CK(cudaEventRecord(h->ev_comp[b], s));
    CK(cudaStreamWaitEvent(h->cs_out, h->ev_comp[b], 0));
    CK(cudaMemcpy2DAsync(C + n1 * j0, 4 * (size_t)(n1 * n4), dC[b], 4 * (size_t)(n1 * wi), 4 * (size_t)(n1 * wi),
                         (size_t)n3, cudaMemcpyDeviceToHost, h->cs_out));
    CK(cudaEventRecord(h->ev_out[b], h->cs_out));
  }
  CK(cudaStreamWaitEvent(s, h->ev_out[0], 0));
  CK(cudaStreamWaitEvent(s, h->ev_out[1], 0));
  CK(cudaStreamSynchronize(s));
  return TPROD_OK;
}

template <typename T>
int host_call(const T* A, const T* B, T* C, int64_t n1, int64_t n2, int64_t n3, int64_t n4,
                     void* stream, tprod_handle h) {
  int st = check_call(h, A, B, C, n1, n2, n3, n4);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  if (sizeof(T) == 4) {
    // pipeline when B is large enough to amortise chunking: 8 to 32 chunks of ~256 MB of B (the
    // tail -- the last chunk's compute and copy-out -- shrinks with the chunk; measured on config 5:
    // 8 chunks 295 ms, 16 279 ms, 32 275 ms against 246 ms of host-to-device copy)
    const double bB = 4.0 * n2 * n4 * n3;
    int64_t chunks = std::min<int64_t>(32, std::max<int64_t>(8, (int64_t)(bB / 256e6 + 0.5)));
    if (const char* e = getenv("TPROD_HOST_CHUNKS")) chunks = std::max(2, atoi(e));   // tuning override
    int64_t w = (n4 + chunks - 1) / chunks;
    if (bB >= 32e6 && n4 >= 4)
      return host_call_f32_pipelined((const float*)A, (const float*)B, (float*)C, n1, n2, n3, n4,
                                     (cudaStream_t)stream, h, w);
  }
  cudaStream_t s = (cudaStream_t)stream;
  size_t bA = sizeof(T) * (size_t)(n1 * n2 * n3), bB = sizeof(T) * (size_t)(n2 * n4 * n3),
         bC = sizeof(T) * (size_t)(n1 * n4 * n3);
  if ((st = ensure_hbuf(h, 0, bA, s)) || (st = ensure_hbuf(h, 1, bB, s)) || (st = ensure_hbuf(h, 2, bC, s))) return st;
  CK(cudaMemcpyAsync(h->hbuf[0], A, bA, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(h->hbuf[1], B, bB, cudaMemcpyHostToDevice, s));
  if (sizeof(T) == 4)
    st = run_f32(h, (const float*)h->hbuf[0], (const float*)h->hbuf[1], (float*)h->hbuf[2], n1, n2, n3, n4, s);
  else
    st = run_f64(h, (const double*)h->hbuf[0], (const double*)h->hbuf[1], (double*)h->hbuf[2], n1, n2, n3, n4, s);
  if (st) return st;
  CK(cudaMemcpyAsync(C, h->hbuf[2], bC, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return TPROD_OK;
}

template <typename T>
int tran_impl(const T* A, T* At, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h) {
  if (!h || !A || !At) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, 1);
  if (st) return st;
  const size_t b = sizeof(T) * (size_t)(n1 * n2 * n3);
  if (overlaps(A, b, At, b)) return TPROD_EALIAS;
  if (n3 > 65535) return TPROD_EUNSUPPORTED;
  CK(cudaSetDevice(h->device));
  launch_tran<T>(A, At, n1, n2, n3, (cudaStream_t)stream);
  h->last_launches = 1;
  return launch_status();
}
template <typename T>
int teye_impl(T* I, int64_t n, int64_t n3, void* stream, tprod_handle h) {
  if (!h || !I) return TPROD_EINVAL;
  int st = validate_dims(n, n, n3, 1);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  if (launch_teye<T>(I, n, n3, (cudaStream_t)stream)) return TPROD_ECUDA;
  h->last_launches = 1;
  return launch_status();
}
// Forward transform of an n1 x n2 x n3 tensor decoded to fp32 spectral planes re/im [f][q][p]
// (the production K1 kernels), into the handle workspace; `extra` bytes are reserved after the
// planes (returned in *extra_ptr).  Used by t-SVT / t-SVD scalars.
int spectral_planes(tprod_ctx* h, const float* Y, int64_t n1, int64_t n2, int64_t n3, size_t extra, float** re,
                    float** im, void** extra_ptr, Twiddles32* Tout, cudaStream_t s) {
  int st;
  const int64_t hh = h_slices(n3), ld = round_up(n1, 8), mn = n1 * n2;
  int f1 = 0, f2 = 0;
  fourstep_factors(n3, &f1, &f2);
  const size_t wb = f1 ? 4 * (size_t)(n1 * n2 * n3) : 0;
  size_t o = 0;
  const size_t off_max = o;  o = align_up(o + 4 * (size_t)n1, 1024);
  const size_t off_u = o;    o = align_up(o + 4 * (size_t)n1, 1024);
  const size_t off_sp = o;   o = align_up(o + 2 * (size_t)(hh * NPLANES * n2 * ld), 1024);
  const size_t off_re = o;   o = align_up(o + 4 * (size_t)(2 * hh * mn), 1024);
  const size_t off_x = o;    o = align_up(o + extra, 1024);
  const size_t off_w = o;    o = align_up(o + wb, 1024);
  if ((st = ensure_ws(h, o, s)) || (st = poison_ws(h, o, s))) return st;
  char* ws = (char*)h->ws;
  Twiddles32 T;
  if ((st = get_twiddles32(h, (int)n3, &T))) return st;
  T.staged = h->transform != 1;
  T.cluster = h->transform == 3;
  T.tc = 0;   // NEXT rows decode the spectrum to fp32: the FFT forward kernels (more accurate than 3xTF32)
  T.scratch = f1 ? (float*)(ws + off_w) : nullptr;
  T.scratch_bytes = wb;
  unsigned* mx = (unsigned*)(ws + off_max);
  float* u = (float*)(ws + off_u);
  __half* sp = (__half*)(ws + off_sp);
  *re = (float*)(ws + off_re);
  *im = *re + hh * mn;
  *extra_ptr = ws + off_x;
  CK(cudaMemsetAsync(mx, 0, 4 * (size_t)n1, s));
  launch_absmax(Y, n1, n2, n3, 0, mx, s);
  launch_fwd_split(Y, n1, n2, n3, 0, mx, T, sp, ld, u, h->num_sms, s);
  launch_decode_split(sp, ld, n1, n2, n3, 0, u, *re, *im, s);
  // Eq. (8): the DC slice and (n3 even) the Nyquist slice are real; their imaginary planes are set
  // to exact zeros, so the per-slice SVD of those slices stays real (R19)
  CK(cudaMemsetAsync(*im, 0, 4 * (size_t)mn, s));
  if (n3 % 2 == 0) CK(cudaMemsetAsync(*im + (n3 / 2) * mn, 0, 4 * (size_t)mn, s));
  *Tout = T;
  return launch_status();
}

}  // namespace

// ====================================================================== exported C ABI
extern "C" {

int tprod_create(int device, tprod_handle* out) {
  if (!out) return TPROD_EINVAL;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return TPROD_ECUDA; }
  if (device < 0 || device >= n) return TPROD_EINVAL;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0) return TPROD_EUNSUPPORTED;   // sm_100a binary only
  CK(cudaSetDevice(device));
  int* status = nullptr;
  CK(cudaMalloc(&status, sizeof(int)));
  CK(cudaMemset(status, 0, sizeof(int)));
  int* done = nullptr;
  if (cudaMalloc(&done, sizeof(int) * (OVERLAP_COUNTERS + 1)) != cudaSuccess) {   // + the K3 work counter
    cudaFree(status);
    return TPROD_ECUDA;
  }
  tprod_ctx* h = new tprod_ctx;
  h->done = done;
  h->device = device;
  h->num_sms = prop.multiProcessorCount;
  h->status = status;
  fork_ready(h);                      // side stream + events now, never inside a stream capture
  *out = h;
  return TPROD_OK;
}

int tprod_destroy(tprod_handle h) {
  if (!h) return TPROD_EINVAL;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  if (h->comm && nccl().ok) nccl().CommDestroy((ncclComm_t)h->comm);
  for (int i = 0; i < 5; ++i) if (h->ev[i]) cudaEventDestroy(h->ev[i]);
  for (auto& kv : h->tw32) cudaFree(kv.second);
  for (auto& kv : h->st32) cudaFree(kv.second);
  for (auto& kv : h->tw64) cudaFree(kv.second);
  for (int i = 0; i < 3; ++i) if (h->hbuf[i]) cudaFree(h->hbuf[i]);
  if (h->prep.buf) cudaFree(h->prep.buf);
  if (h->prep_host.buf) cudaFree(h->prep_host.buf);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_in[i]) cudaEventDestroy(h->ev_in[i]);
    if (h->ev_comp[i]) cudaEventDestroy(h->ev_comp[i]);
    if (h->ev_out[i]) cudaEventDestroy(h->ev_out[i]);
  }
  if (h->cs_in) cudaStreamDestroy(h->cs_in);
  if (h->cs_out) cudaStreamDestroy(h->cs_out);
  clear_graphs(h);
  if (h->cap) cudaStreamDestroy(h->cap);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ws) cudaFree(h->ws);
  if (h->status) cudaFree(h->status);
  if (h->done) cudaFree(h->done);
  for (void* p : h->retired) cudaFree(p);
  delete h;
  return TPROD_OK;
}

int tprod_f32(const float* A, const float* B, float* C, int64_t n1, int64_t n2, int64_t n3,
              int64_t n4, void* stream, tprod_handle h) {
  int st = check_call(h, A, B, C, n1, n2, n3, n4);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  return run_f32(h, A, B, C, n1, n2, n3, n4, (cudaStream_t)stream);
}

int tprod_f64(const double* A, const double* B, double* C, int64_t n1, int64_t n2, int64_t n3,
              int64_t n4, void* stream, tprod_handle h) {
  int st = check_call(h, A, B, C, n1, n2, n3, n4);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  return run_f64(h, A, B, C, n1, n2, n3, n4, (cudaStream_t)stream);
}

int tprod_f32_host(const float* A, const float* B, float* C, int64_t n1, int64_t n2, int64_t n3,
                   int64_t n4, void* stream, tprod_handle h) {
  return host_call(A, B, C, n1, n2, n3, n4, stream, h);
}

int tprod_f64_host(const double* A, const double* B, double* C, int64_t n1, int64_t n2, int64_t n3,
                   int64_t n4, void* stream, tprod_handle h) {
  return host_call(A, B, C, n1, n2, n3, n4, stream, h);
}

int tprod_prepare_a_f32(const float* A, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h) {
  if (!h || !A) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, 1);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  return prepare_into(h, h->prep, A, n1, n2, n3, (cudaStream_t)stream);
}

int tprod_f32_prepared(const float* B, float* C, int64_t n4, void* stream, tprod_handle h) {
  if (!h || !B || !C || !h->prep.valid) return TPROD_EINVAL;
  const PreparedA& P = h->prep;
  int st = validate_dims(P.n1, P.n2, P.n3, n4);
  if (st) return st;
  if (overlaps(C, 4 * (size_t)(P.n1 * n4 * P.n3), B, 4 * (size_t)(P.n2 * n4 * P.n3))) return TPROD_EALIAS;
  CK(cudaSetDevice(h->device));
  return run_f32(h, nullptr, B, C, P.n1, P.n2, P.n3, n4, (cudaStream_t)stream, &P);
}

int tprod_release_a(tprod_handle h) {
  if (!h) return TPROD_EINVAL;
  if (h->prep.buf) {                                 // synchronous by contract (include/tprod.h)
    CK(cudaSetDevice(h->device));
    CK(cudaDeviceSynchronize());
    cudaFree(h->prep.buf);
    h->async_buf.erase(h->prep.buf);
  }
  h->prep = PreparedA();
  return TPROD_OK;
}

int tprod_tran_f32(const float* A, float* At, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h) {
  return tran_impl(A, At, n1, n2, n3, stream, h);
}
int tprod_tran_f64(const double* A, double* At, int64_t n1, int64_t n2, int64_t n3, void* stream, tprod_handle h) {
  return tran_impl(A, At, n1, n2, n3, stream, h);
}

int tprod_teye_f32(float* I, int64_t n, int64_t n3, void* stream, tprod_handle h) {
  return teye_impl(I, n, n3, stream, h);
}
int tprod_teye_f64(double* I, int64_t n, int64_t n3, void* stream, tprod_handle h) {
  return teye_impl(I, n, n3, stream, h);
}

int tprod_tinv_f32(const float* A, float* X, int64_t n, int64_t n3, void* stream, tprod_handle h) {
  if (!h || !A || !X) return TPROD_EINVAL;
  int st = validate_dims(n, n, n3, 1);
  if (st) return st;
  if (n > 8192) return TPROD_EUNSUPPORTED;
  const size_t b = 4 * (size_t)(n * n * n3);
  if (overlaps(A, b, X, b)) return TPROD_EALIAS;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t hh = h_slices(n3), ld = round_up(n, 8), nn = n * n;
  int f1 = 0, f2 = 0;
  fourstep_factors(n3, &f1, &f2);
  size_t o = 0;
  const size_t off_flag = o; o = align_up(o + 16, 1024);                    // singular flag, max entry
  const size_t off_max = o;  o = align_up(o + 4 * (size_t)n, 1024);
  const size_t off_u = o;    o = align_up(o + 4 * (size_t)n, 1024);
  const size_t off_sp = o;   o = align_up(o + 2 * (size_t)(hh * NPLANES * n * ld), 1024);
  const size_t off_re = o;   o = align_up(o + 4 * (size_t)(4 * hh * nn), 1024);  // re, im, xre, xim
  const size_t off_w = o;    o = align_up(o + (f1 ? b : 0), 1024);
  const bool small = tinv_supported(n);                                     // n <= 96: shared-memory kernel
  const size_t off_gj = o;   o = align_up(o + (small ? 0 : gj_workspace_bytes(n, hh)), 1024);
  if ((st = ensure_ws(h, o, s)) || (st = poison_ws(h, o, s))) return st;
  char* ws = (char*)h->ws;
  Twiddles32 T;
  if ((st = get_twiddles32(h, (int)n3, &T))) return st;
  T.staged = h->transform != 1;
  T.cluster = h->transform == 3;
  T.tc = 0;   // NEXT rows decode the spectrum to fp32: the FFT forward kernels (more accurate than 3xTF32)
  T.scratch = f1 ? (float*)(ws + off_w) : nullptr;
  T.scratch_bytes = f1 ? b : 0;
  int* flag = (int*)(ws + off_flag);
  unsigned* amax = (unsigned*)(ws + off_flag + 4);
  unsigned* mx = (unsigned*)(ws + off_max);
  float* u = (float*)(ws + off_u);
  __half* sp = (__half*)(ws + off_sp);
  float* re = (float*)(ws + off_re);
  float* im = re + hh * nn;
  float* xre = im + hh * nn;
  float* xim = xre + hh * nn;
  CK(cudaMemsetAsync(ws + off_flag, 0, 16, s));
  CK(cudaMemsetAsync(mx, 0, 4 * (size_t)n, s));
  launch_absmax(A, n, n, n3, 0, mx, s);                                      // row scales
  launch_fwd_split(A, n, n, n3, 0, mx, T, sp, ld, u, h->num_sms, s);         // Alg. 1 step 1
  launch_decode_split(sp, ld, n, n, n3, 0, u, re, im, s);                    // fp32 planes [f][q][p]
  launch_absmax_planes(re, im, hh * nn, amax, s);
  const float rtol = (float)n * 9.5367431640625e-07f;                        // n * 2^-20
  // synchronous checks: this call's own flag, read back below; else the handle's status word
  int* sflag = h->sync_checks ? flag : h->status;
  if (small) {
    if (launch_slice_inverse(re, im, xre, xim, n, hh, nn, rtol, amax, sflag, s)) return TPROD_ECUDA;
  } else {
    if (launch_slice_inverse_large(re, im, xre, xim, n, hh, nn, rtol, amax, sflag, ws + off_gj, s)) return TPROD_ECUDA;
  }
  launch_inv_f32(xre, xim, n, nn, n, n, n3, T, OutUnscale{}, X, h->num_sms, s);            // fill + inverse DFT
  if ((st = launch_status())) return st;
  h->last_launches = small ? 7 : 8 + 2 * n;
  if (!h->sync_checks) return TPROD_OK;
  int host_flag = 0;
  CK(cudaMemcpyAsync(&host_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return host_flag ? TPROD_ESINGULAR : TPROD_OK;
}

int tprod_tsvt_f32(const float* Y, float* X, int64_t n1, int64_t n2, int64_t n3, float tau, void* stream,
                   tprod_handle h) {
  if (!h || !Y || !X || !(tau >= 0.f)) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, 1);
  if (st) return st;
  const size_t b = 4 * (size_t)(n1 * n2 * n3);
  if (overlaps(Y, b, X, b)) return TPROD_EALIAS;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t hh = h_slices(n3), mn = n1 * n2;
  // slices up to 64 x 64: one CTA per slice, Jacobi in shared memory; larger: blocked Jacobi with the
  // slices in the workspace (tsvt_block.cu)
  const bool small = svt_supported(n1, n2);
  const size_t wbytes = align_up(4 * (size_t)(2 * hh * mn), 1024);
  const size_t extra_bytes = wbytes + (small ? 0 : bj_workspace_bytes(n1, n2, hh));
  if (!small && std::min(n1, n2) > 65535) return TPROD_EUNSUPPORTED;
  float *re, *im;
  void* extra;
  Twiddles32 T;
  if ((st = spectral_planes(h, Y, n1, n2, n3, extra_bytes, &re, &im, &extra, &T, s))) return st;  // Alg. 3 step 1
  float* wre = (float*)extra;
  float* wim = wre + hh * mn;
  if (small) {
    if (launch_slice_svt(re, im, wre, wim, n1, n2, hh, mn, tau, h->status, s)) return TPROD_ECUDA;   // step 2
  } else {
    BjOut o{};
    o.tau = tau;
    o.wre = wre;
    o.wim = wim;
    if (launch_block_svd(re, im, n1, n2, hh, mn, BJ_SVT, o, (char*)extra + wbytes, h->status, s)) return TPROD_ECUDA;
  }
  launch_inv_f32(wre, wim, n1, mn, n1, n2, n3, T, OutUnscale{}, X, h->num_sms, s);         // step 2b + 3
  h->last_launches = 5;
  return launch_status();
}

int tprod_tsvd_f32(const float* A, float* U, float* S, float* V, int64_t n1, int64_t n2, int64_t n3, void* stream,
                   tprod_handle h) {
  if (!h || !A || !U || !S || !V) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, 1);
  if (st) return st;
  const bool small = svt_supported(n1, n2);
  if (!small && std::min(n1, n2) > 65535) return TPROD_EUNSUPPORTED;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t hh = h_slices(n3), r = std::min(n1, n2);
  const int64_t nu = n1 * r, ns = r * r, nv = n2 * r;
  float *re, *im;
  void* extra;
  Twiddles32 T;
  const size_t fbytes = align_up(4 * (size_t)(hh * (2 * nu + 2 * ns + 2 * nv)), 1024);
  const size_t ex = fbytes + (small ? 0 : bj_workspace_bytes(n1, n2, hh));
  if ((st = spectral_planes(h, A, n1, n2, n3, ex, &re, &im, &extra, &T, s))) return st;   // Alg. 2 step 1
  float* ure = (float*)extra;
  float* uim = ure + hh * nu;
  float* sre = uim + hh * nu;
  float* sim = sre + hh * ns;
  float* vre = sim + hh * ns;
  float* vim = vre + hh * nv;
  CK(cudaMemsetAsync(sim, 0, 4 * (size_t)(hh * ns), s));                                  // S-bar is real
  if (small) {
    if (launch_slice_svd_factors(re, im, n1, n2, hh, n1 * n2, ure, uim, sre, vre, vim, h->status, s))
      return TPROD_ECUDA;                                                                  // step 2
  } else {
    BjOut o{};
    o.ure = ure;
    o.uim = uim;
    o.sre = sre;
    o.vre = vre;
    o.vim = vim;
    if (launch_block_svd(re, im, n1, n2, hh, n1 * n2, BJ_FACTORS, o, (char*)extra + fbytes, h->status, s))
      return TPROD_ECUDA;
  }
  // step 2b + 3: conjugate fill + inverse DFT of each factor (S-bar's copy rule = conj of a real slice)
  launch_inv_f32(ure, uim, n1, nu, n1, r, n3, T, OutUnscale{}, U, h->num_sms, s);
  launch_inv_f32(sre, sim, r, ns, r, r, n3, T, OutUnscale{}, S, h->num_sms, s);
  launch_inv_f32(vre, vim, n2, nv, n2, r, n3, T, OutUnscale{}, V, h->num_sms, s);
  h->last_launches = 8;
  return launch_status();
}

int tprod_tsvd_full_f32(const float* A, float* U, float* S, float* V, int64_t n1, int64_t n2, int64_t n3,
                        void* stream, tprod_handle h) {
  if (!h || !A || !U || !S || !V) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, 1);
  if (st) return st;
  if (std::max(n1, n2) > 65535) return TPROD_EUNSUPPORTED;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t hh = h_slices(n3);
  const int64_t nu = n1 * n1, ns = n1 * n2, nv = n2 * n2;
  float *re, *im;
  void* extra;
  Twiddles32 T;
  const size_t fbytes = align_up(4 * (size_t)(hh * (2 * nu + 2 * ns + 2 * nv)), 1024);
  const size_t ex = fbytes + bj_workspace_bytes(n1, n2, hh, true);
  if ((st = spectral_planes(h, A, n1, n2, n3, ex, &re, &im, &extra, &T, s))) return st;   // Alg. 2 step 1
  float* ure = (float*)extra;
  float* uim = ure + hh * nu;
  float* sre = uim + hh * nu;
  float* sim = sre + hh * ns;
  float* vre = sim + hh * ns;
  float* vim = vre + hh * nv;
  CK(cudaMemsetAsync(sim, 0, 4 * (size_t)(hh * ns), s));                                  // S-bar is real
  BjOut o{};
  o.ure = ure;
  o.uim = uim;
  o.sre = sre;
  o.vre = vre;
  o.vim = vim;
  // step 2: full SVD of every spectral slice (blocked Jacobi for all sizes; the left basis of the
  // processed slice completed to max(n1, n2) orthonormal columns)
  if (launch_block_svd(re, im, n1, n2, hh, n1 * n2, BJ_FACTORS_FULL, o, (char*)extra + fbytes, h->status, s))
    return TPROD_ECUDA;
  launch_inv_f32(ure, uim, n1, nu, n1, n1, n3, T, OutUnscale{}, U, h->num_sms, s);          // step 2b + 3
  launch_inv_f32(sre, sim, n1, ns, n1, n2, n3, T, OutUnscale{}, S, h->num_sms, s);
  launch_inv_f32(vre, vim, n2, nv, n2, n2, n3, T, OutUnscale{}, V, h->num_sms, s);
  h->last_launches = 8;
  return launch_status();
}

int tprod_tsvd_values_f32(const float* A, int64_t n1, int64_t n2, int64_t n3, float rtol, float* out, void* stream,
                          tprod_handle h) {
  if (!h || !A || !out || !(rtol >= 0.f)) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, 1);
  if (st) return st;
  const bool small = svt_supported(n1, n2);
  if (!small && std::min(n1, n2) > 65535) return TPROD_EUNSUPPORTED;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t hh = h_slices(n3), r = std::min(n1, n2);
  float *re, *im;
  void* extra;
  Twiddles32 T;
  const size_t svb = align_up(8 * (size_t)(hh * r), 1024);
  const size_t ex = svb + (small ? 0 : bj_workspace_bytes(n1, n2, hh));
  if ((st = spectral_planes(h, A, n1, n2, n3, ex, &re, &im, &extra, &T, s))) return st;  // Alg. 2 step 1
  if (small) {
    if (launch_tsvd_values(re, im, n1, n2, hh, n3, n1 * n2, (double*)extra, rtol, out, h->status, s))
      return TPROD_ECUDA;
  } else {
    BjOut o{};
    o.sv = (double*)extra;
    if (launch_block_svd(re, im, n1, n2, hh, n1 * n2, BJ_VALUES, o, (char*)extra + svb, h->status, s) ||
        launch_tsvd_reduce((double*)extra, r, hh, n3, rtol, out, s))
      return TPROD_ECUDA;
  }
  h->last_launches = 5;
  return launch_status();
}

int tprod_workspace_bytes(int64_t n1, int64_t n2, int64_t n3, int64_t n4, int dtype, size_t* out) {
  if (!out) return TPROD_EINVAL;
  int st = validate_dims(n1, n2, n3, n4);
  if (st) return st;
  if (dtype == TPROD_DTYPE_F32) *out = layout32(n1, n2, n3, n4).total;
  else if (dtype == TPROD_DTYPE_F64) *out = layout64(n1, n2, n3, n4).total;
  else return TPROD_EINVAL;
  return TPROD_OK;
}

const char* tprod_strerror(int status) {
  switch (status) {
    case TPROD_OK: return "ok";
    case TPROD_EINVAL: return "invalid argument (dimension < 1, NULL pointer, size overflow or bad handle)";
    case TPROD_EALIAS: return "output C overlaps input A or B (in-place t-product is not supported)";
    case TPROD_ENOMEM: return "device memory allocation failed";
    case TPROD_ECUDA: return "CUDA runtime or kernel launch error";
    case TPROD_ENCCL: return "NCCL unavailable or an NCCL call failed";
    case TPROD_EUNSUPPORTED: return "unsupported device or shape (requires sm_100 / B200)";
    case TPROD_ENOWORLD: return "no NCCL world: call tprod_set_world first";
    case TPROD_ESINGULAR: return "singular tensor: a spectral slice has no inverse to working precision";
    default: return "unknown tprod status";
  }
}

int tprod_last_launch_count(tprod_handle h, int64_t* out) {
  if (!h || !out) return TPROD_EINVAL;
  *out = h->last_launches;
  return TPROD_OK;
}

int tprod_nccl_unique_id(void* out) {
  if (!out) return TPROD_EINVAL;
  if (!nccl().ok) return TPROD_ENCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return TPROD_ENCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  memcpy(out, &id, sizeof(id));
  return TPROD_OK;
}

int tprod_set_world(tprod_handle h, int rank, int world, const void* uid) {
  if (!h || !uid || world < 1 || rank < 0 || rank >= world) return TPROD_EINVAL;
  if (!nccl().ok) return TPROD_ENCCL;
  CK(cudaSetDevice(h->device));
  if (h->comm) { nccl().CommDestroy((ncclComm_t)h->comm); h->comm = nullptr; }
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclComm_t comm;
  if (nccl().CommInitRank(&comm, world, id, rank) != ncclSuccess) return TPROD_ENCCL;
  h->comm = comm;
  h->rank = rank;
  h->world = world;
  return TPROD_OK;
}

static int bcast(tprod_handle h, void* buf, int64_t count, ncclDataType_t dt, int root, void* stream) {
  if (!h || !buf || count < 0) return TPROD_EINVAL;
  if (!h->comm) return TPROD_ENOWORLD;
  if (root < 0 || root >= h->world) return TPROD_EINVAL;
  CK(cudaSetDevice(h->device));
  if (nccl().Broadcast(buf, buf, (size_t)count, dt, root, (ncclComm_t)h->comm, (cudaStream_t)stream) != ncclSuccess)
    return TPROD_ENCCL;
  return TPROD_OK;
}

int tprod_bcast_f32(tprod_handle h, float* buf, int64_t count, int root, void* stream) {
  return bcast(h, buf, count, ncclFloat32, root, stream);
}
int tprod_bcast_f64(tprod_handle h, double* buf, int64_t count, int root, void* stream) {
  return bcast(h, buf, count, ncclFloat64, root, stream);
}

int tprod_dft_f32(const float* X, float* Xre, float* Xim, int64_t p, int64_t q, int64_t n3,
                  int role, void* stream, tprod_handle h) {
  if (!h || !X || !Xre || !Xim || (role != 0 && role != 1)) return TPROD_EINVAL;
  int st = validate_dims(p, q, n3, 1);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  int64_t hh = h_slices(n3), ld = round_up(p, 8);
  int64_t nmax = role == 0 ? p : q;
  size_t off_u = align_up(4 * (size_t)nmax, 1024);
  size_t off_sp = off_u + align_up(4 * (size_t)nmax, 1024);
  int f1 = 0, f2 = 0;
  fourstep_factors(n3, &f1, &f2);
  const size_t w_bytes = f1 ? 4 * (size_t)(p * q * n3) : 0;            // four-step intermediate
  const size_t off_w = align_up(off_sp + 2 * (size_t)(hh * NPLANES * q * ld), 1024);
  if ((st = ensure_ws(h, off_w + w_bytes, s)) || (st = poison_ws(h, off_w + w_bytes, s))) return st;
  Twiddles32 T;
  if ((st = get_twiddles32(h, (int)n3, &T))) return st;
  T.staged = h->transform != 1;
  T.cluster = h->transform == 3;
  T.tc = h->transform == 2;
  T.scratch = w_bytes ? (float*)((char*)h->ws + off_w) : nullptr;
  T.scratch_bytes = w_bytes;
  unsigned* mx = (unsigned*)h->ws;
  float* u = (float*)((char*)h->ws + off_u);
  __half* sp = (__half*)((char*)h->ws + off_sp);
  CK(cudaMemsetAsync(mx, 0, 4 * (size_t)nmax, s));
  launch_absmax(X, p, q, n3, role, mx, s);
  launch_fwd_split(X, p, q, n3, role, mx, T, sp, ld, u, h->num_sms, s);
  launch_decode_split(sp, ld, p, q, n3, role, u, Xre, Xim, s);
  h->last_launches = 3;
  return launch_status();
}

int tprod_idft_f32(const float* Xre, const float* Xim, float* X, int64_t p, int64_t q, int64_t n3,
                   void* stream, tprod_handle h) {
  if (!h || !Xre || !Xim || !X) return TPROD_EINVAL;
  int st = validate_dims(p, q, n3, 1);
  if (st) return st;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  Twiddles32 T;
  if ((st = get_twiddles32(h, (int)n3, &T))) return st;
  launch_inv_f32(Xre, Xim, p, p * q, p, q, n3, T, OutUnscale{}, X, h->num_sms, s);
  h->last_launches = 1;
  return launch_status();
}

int tprod_set_option(tprod_handle h, int option, int64_t value) {
  if (!h) return TPROD_EINVAL;
  switch (option) {
    case TPROD_OPT_ENGINE:
      if (value != 0 && value != 1) return TPROD_EINVAL;
      h->engine = (int)value;
      return TPROD_OK;
    case TPROD_OPT_TIMING:
      if (value != 0 && value != 1) return TPROD_EINVAL;
      if (value && !h->ev[0]) {
        CK(cudaSetDevice(h->device));
        for (int i = 0; i < 5; ++i) CK(cudaEventCreate(&h->ev[i]));
      }
      h->timing = value != 0;
      return TPROD_OK;
    case TPROD_OPT_GEMM_CLUSTER:
      if (value < 0 || value > 4) return TPROD_EINVAL;
      h->force_cn = (int)value;
      return TPROD_OK;
    case TPROD_OPT_TRANSFORM:
      if (value < 0 || value > 3) return TPROD_EINVAL;
      h->transform = (int)value;
      return TPROD_OK;
    case TPROD_OPT_GEMM_BN:
      if (value != 0 && value != 64 && value != 128) return TPROD_EINVAL;
      h->force_bn = (int)value;
      return TPROD_OK;
    case TPROD_OPT_GRAPHS:
      if (value != 0 && value != 1) return TPROD_EINVAL;
      h->graphs = value != 0;
      return TPROD_OK;
    case TPROD_OPT_POISON:
      if (value != 0 && value != 1) return TPROD_EINVAL;
      h->poison = value != 0;
      return TPROD_OK;
    case TPROD_OPT_SYNC_CHECKS:
      if (value != 0 && value != 1) return TPROD_EINVAL;
      h->sync_checks = value != 0;
      return TPROD_OK;
    case TPROD_OPT_OVERLAP:
      if (value < 0 || value > 2) return TPROD_EINVAL;
      h->overlap = value != 0;
      h->overlap_stream = value == 1;
      return TPROD_OK;
    case TPROD_OPT_FUSED_SCALES:
      if (value != 0 && value != 1) return TPROD_EINVAL;
      h->fused_scales = value != 0;
      return TPROD_OK;
    default:
      return TPROD_EINVAL;
  }
}

int tprod_status(tprod_handle h, void* stream, int* bits) {
  if (!h || !bits) return TPROD_EINVAL;
  CK(cudaSetDevice(h->device));
  cudaStream_t s = (cudaStream_t)stream;
  int v = 0;
  CK(cudaMemcpyAsync(&v, h->status, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaMemsetAsync(h->status, 0, sizeof(int), s));
  CK(cudaStreamSynchronize(s));
  *bits = v;
  return TPROD_OK;
}

int tprod_last_stage_ms(tprod_handle h, float* out) {
  if (!h || !out || !h->timed_last) return TPROD_EINVAL;
  CK(cudaEventSynchronize(h->ev[4]));
  if (h->forked_last) {               // concurrent A / B chains: K0 + K1 as one stage (tprod.h)
    CK(cudaEventElapsedTime(out, h->ev[0], h->ev[2]));
    out[1] = 0.f;
  } else {
    for (int i = 0; i < 2; ++i) CK(cudaEventElapsedTime(out + i, h->ev[i], h->ev[i + 1]));
  }
  if (h->overlapped_last) {           // K2 and K3 overlapped: one stage (tprod.h)
    CK(cudaEventElapsedTime(out + 2, h->ev[2], h->ev[4]));
    out[3] = 0.f;
  } else {
    for (int i = 2; i < 4; ++i) CK(cudaEventElapsedTime(out + i, h->ev[i], h->ev[i + 1]));
  }
  return TPROD_OK;
}

}  // extern "C"
