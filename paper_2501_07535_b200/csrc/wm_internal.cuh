// Host-side internals shared by the library's translation units: error
// channel, small host bignum helpers for parameter setup, the field and plan
// objects, and the limb-count dispatch tables.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/widemod_b200.h"
#include "wm_limb.cuh"

namespace wm {

// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define WM_CUDA_TRY(expr)                                  \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return ::wm::cuda_fail(_e, #expr); \
  } while (0)

// After a kernel launch: report launch-configuration errors synchronously.
#define WM_LAUNCH_CHECK(what)                              \
  do {                                                     \
    cudaError_t _e = cudaGetLastError();                   \
    if (_e != cudaSuccess) return ::wm::cuda_fail(_e, what); \
  } while (0)

// cudaFuncSetAttribute acts on the current device: attribute setup done once
// per (call site, device).  Returns true the first time for the current device.
inline bool first_on_device(std::atomic<uint64_t> &mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return true;
  const uint64_t bit = 1ull << (dev & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

// ------------------------------------------------------------------ limb sets
// Limb counts compiled into the library.  K = ceil(bits/32).
#ifndef WM_BLAS_KS
#define WM_BLAS_KS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(24) X(32)
#endif
// Full-width (Montgomery) fields: the common curve / FHE sizes.
#ifndef WM_MONT_KS
#define WM_MONT_KS(X) X(1) X(2) X(4) X(8) X(12) X(16) X(24) X(32)
#endif
#ifndef WM_NTT_KS
#define WM_NTT_KS(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(24) X(32)
#endif

bool blas_supports(int K);
bool ntt_supports(int K);
bool mont_supports(int K);

// ------------------------------------------------------------------ host bignum
using Big = std::vector<uint32_t>;  // little-endian limbs, fixed length
int big_bitlen(const Big &a);
Big big_shl(const Big &a, int s, int limbs);          // (a << s) truncated to limbs
bool big_ge(const Big &a, const Big &b);               // same length
void big_sub_inplace(Big &a, const Big &b);            // a -= b, same length, a >= b
Big big_resize(const Big &a, int limbs);
// floor(2^e / d) truncated to `limbs` limbs (binary long division).
Big big_pow2_div(int e, const Big &d, int limbs);
// (a * 2^e) mod q, a < q, K = q.size() limbs.
Big big_shl_mod(const Big &a, int e, const Big &q);
// Montgomery form a * 2^(32K) mod q.
inline Big to_mont(const Big &a, const Big &q) { return big_shl_mod(a, 32 * (int)q.size(), q); }

// ------------------------------------------------------------------ host pipeline
// Streams, events and device staging slots of a host-buffer pipeline
// (wm_ntt_host, wm_blas_host): h2d, d2h, then kComp compute streams; chunks
// round-robin over the compute streams and over kSlots staging slots.
// Created on first use, guarded by `mu` (one pipelined call at a time per
// owner object).
struct HostPipe {
  static constexpr int kComp = 4;
  static constexpr int kStreams = 2 + kComp;
  static constexpr int kSlots = 8;
  std::mutex mu;
  bool ready = false;
  cudaStream_t hs[kStreams] = {};
  cudaEvent_t ev_in[kSlots] = {}, ev_comp[kSlots] = {}, ev_out[kSlots] = {};
  cudaEvent_t ev_entry = nullptr, ev_done = nullptr;
  void *slot_mem[kSlots] = {};
  int64_t slot_bytes = 0;
  int ensure(int64_t bytes);  // streams/events created, every slot >= bytes
  void release();
};

// ------------------------------------------------------------------ objects
}  // namespace wm

struct wm_field {
  bool karatsuba = false;  // vmul/axpy use the Karatsuba full product
  bool mont = false;       // full-width modulus, Montgomery arithmetic (WM_FIELD_MONTGOMERY)
  uint32_t qinv = 0;       // mont: -q^-1 mod 2^32
  wm::Big r2;              // mont: 2^(64K) mod q
  int bits = 0;
  int K = 0;
  int s = 0;
  wm::Big q, qn, qn2, nqn, mu8;  // K limbs each
  // special form q = 2^m - pm_c (pm_c < 2^32, 72 <= m, 4 <= 32K - m <= 31):
  // vmul/axpy/NTT products reduce by two folds (mul_pm_lazy) unless the field
  // was created with WM_FIELD_BARRETT; the Barrett constants stay valid
  bool pm = false;
  uint32_t pm_c = 0;
  int pm_sh = 0;
  wm::HostPipe host;  // wm_blas_host staging (created on first use)
};

struct wm_pass_plan {
  bool column = false;  // column pass (strided lines) vs row pass (contiguous lines)
  int logL = 0;         // sub-transform size
  int G = 1;            // lines per CTA
  // column pass: line (o, i); read pos = o*RO + t*RT + i; write pos = o*WO + k*WK + i
  // row pass:    line r;      read pos = r*L + t;         write pos = r*WO + k*WK
  int64_t lines_inner = 1, lines_outer = 1;
  int64_t RO = 0, RT = 0, WO = 0, WK = 0;
  // twiddle on output: e = ((i >> SH) * (o*C1 + k*C2) * C3) mod n; C3 == 0: none
  int SH = 0;
  int64_t C1 = 0, C2 = 0, C3 = 0;
  bool scaled_table = false;  // inverse: use the n^-1-scaled table for this pass
  bool scale_out = false;     // inverse one-pass plans: multiply outputs by n^-1
  bool canonical_out = false; // last pass of the transform: [0, 6p) -> [0, p)
  int src = 0, dst = 0;       // 0 = user in/out, 1 = workspace (see plan creation)
};

struct wm_ntt_plan {
  const wm_field *field = nullptr;
  int K = 0;
  int64_t n = 0;
  int logn = 0;
  std::vector<wm_pass_plan> passes;
  // device tables: n entries of (w, w') pairs (2K words each)
  uint32_t *tw_fwd = nullptr, *tw_inv = nullptr, *tw_inv_scaled = nullptr;
  // per-pass twiddle sub-tables as shared-memory images (TMA bulk-copied by the
  // pass kernels): forward images at tw_img + tw_img_off[pass], inverse images
  // tw_img_words_dir words further
  uint32_t *tw_img = nullptr;
  std::vector<size_t> tw_img_off;
  size_t tw_img_words_dir = 0;
  int mode = 0;        // Arith mode: 0 lazy Shoup [0,6p), 1 Montgomery, 2 Shoup [0,4p) (full-width p < 2^(32K-2)),
                       // 3 lazy special-form products [0,6p) (wm_field.pm)
  wm::Big ninv_mont;  // full-width fields: n^-1 R mod p (one-pass inverse scale)
  wm::Big ninv, ninv_sh, np, p2, p3, p4;  // n^-1, floor(n^-1 * 2^32K / p), 2^32K - p, 2p, 3p, 4p
  // internal workspace (used when the caller passes none): uses are
  // stream-ordered through ws_ev (ntt_run_internal)
  std::mutex ws_mu;
  cudaEvent_t ws_ev = nullptr;
  void *ws = nullptr;
  int64_t ws_bytes = 0;
  wm::HostPipe host;  // wm_ntt_host staging (created on first use)
};

namespace wm {
// Device constants of a field (the one place they are packed for kernels).
template <int K>
inline FieldConst<K> field_const(const wm_field *f) {
  FieldConst<K> c;
  for (int j = 0; j < K; ++j) {
    c.q[j] = f->q[j];
    c.qn[j] = f->qn[j];
    c.qn2[j] = f->qn2[j];
    c.nqn[j] = f->nqn[j];
    c.mu8[j] = f->mu8[j];
    c.r2[j] = f->mont ? f->r2[j] : 0u;
  }
  c.s = (uint32_t)f->s;
  c.qinv = f->qinv;
  c.pm_c = f->pm_c;
  c.pm_sh = (uint32_t)f->pm_sh;
  return c;
}

int ntt_mode_for(const wm_field *f);
// Load the kernel images a field's BLAS calls and transforms use (CUDA lazy
// loading synchronises the context on a kernel's first load); best effort.
void preload_ntt(const wm_field *f);
void preload_field(const wm_field *f);
int ntt_run_internal(const wm_ntt_plan *p, bool inverse, const uint32_t *in, uint32_t *out, int64_t batch,
                     void *workspace, cudaStream_t st, const uint32_t *mul_by = nullptr);

}  // namespace wm
