// NTT plans and the C ABI entry points of the transform (host side).  The
// kernels and per-limb-count host templates are in wm_ntt_impl.cuh; see its
// header comment for the design.
#include "wm_ntt_impl.cuh"

namespace wm {
#define WM_EXTERN_INST(k) WM_NTT_INSTANTIATE(extern, k)
WM_NTT_KS(WM_EXTERN_INST)
#undef WM_EXTERN_INST

// Arithmetic mode of a field's transforms: full-width fields with two bits of
// headroom take the Shoup / [0, 4p) path (2), the other full-width fields the
// Montgomery path (1); special-form reference-range fields the two-fold
// products (3), the rest Shoup / [0, 6p) (0).
#ifndef WM_PM_NTT
#define WM_PM_NTT 1
#endif
int ntt_mode_for(const wm_field *f) {
  if (f->mont) return big_bitlen(f->q) <= 32 * f->K - 2 ? 2 : 1;
  return (WM_PM_NTT && f->pm && f->K >= 3) ? 3 : 0;
}

void preload_ntt(const wm_field *f) {
  if (!ntt_supports(f->K)) return;
  const int mode = ntt_mode_for(f);
  switch (f->K) {
#define WM_CASE(k)            \
  case k:                     \
    ntt_preload<k>(mode);     \
    break;
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      break;
  }
}

static int plan_passes(wm_ntt_plan *pl) {
  const int K = pl->K;
  const int logn = pl->logn;
  // largest sub-transform whose line fits in <= 96 KB of shared memory
  int logLmax = 1;
  while (logLmax < 11 && ((size_t)2 << logLmax) * K * 4 <= 96 * 1024) ++logLmax;
  const int P = (logn + logLmax - 1) / logLmax;
  if (P > 3) return fail(WM_EUNSUPPORTED, "transform too long for three passes at this width");
  std::vector<int> sizes(P, logn / P);
  for (int i = 0; i < logn % P; ++i) sizes[i] += 1;
  auto choose_G = [&](int logL, int64_t inner_cap) {
    int64_t words_line = ((int64_t)1 << logL) * K;
    const int64_t tile = K <= 4 ? WM_NTT_TILE_WORDS_SMALL : WM_NTT_TILE_WORDS;  // data words per CTA
    int64_t G = std::max<int64_t>(1, tile / words_line);
    G = std::min<int64_t>(G, 32);
    int64_t g = 1;
    while (g * 2 <= G) g *= 2;
    return (int)std::min<int64_t>(g, inner_cap);
  };
  pl->passes.clear();
  const int64_t n = pl->n;
  if (P == 1) {
    wm_pass_plan a;
    a.column = false;
    a.logL = logn;
    a.G = choose_G(logn, 1 << 20);
    a.lines_inner = 1;
    a.WO = n;
    a.WK = 1;
    a.scale_out = true;
    a.src = 0;
    a.dst = 0;
    pl->passes.push_back(a);
  } else if (P == 2) {
    const int logN2 = sizes[0], logN1 = sizes[1];
    const int64_t N1 = (int64_t)1 << logN1, N2 = (int64_t)1 << logN2;
    wm_pass_plan a;  // N2-point DFTs over j2 (stride N1), twiddle root^(j1*k2)
    a.column = true;
    a.logL = logN2;
    a.G = choose_G(logN2, N1);
    a.lines_inner = N1;
    a.lines_outer = 1;
    a.RO = 0;
    a.RT = N1;
    a.WO = 0;
    a.WK = N1;
    a.SH = 0;
    a.C1 = 0;
    a.C2 = 1;
    a.C3 = 1;
    a.scaled_table = true;
    a.src = 0;
    a.dst = 1;
    wm_pass_plan b;  // N1-point DFTs over contiguous j1, transposing store
    b.column = false;
    b.logL = logN1;
    b.G = choose_G(logN1, 1 << 20);
    b.lines_inner = N2;
    b.WO = 1;
    b.WK = N2;
    b.src = 1;
    b.dst = 0;
    pl->passes.push_back(a);
    pl->passes.push_back(b);
  } else {
    const int logM2 = sizes[0], logM1 = sizes[1], logN1 = sizes[2];
    const int64_t N1 = (int64_t)1 << logN1, M1 = (int64_t)1 << logM1, M2 = (int64_t)1 << logM2;
    const int64_t N2 = M1 * M2;
    wm_pass_plan a;  // M2-point DFTs over b, lines i = j1 + N1*a; twiddle root^(N1*a*c)
    a.column = true;
    a.logL = logM2;
    a.G = choose_G(logM2, N1 * M1);
    a.lines_inner = N1 * M1;
    a.lines_outer = 1;
    a.RT = N1 * M1;
    a.WK = N1 * M1;
    a.SH = logN1;
    a.C1 = 0;
    a.C2 = 1;
    a.C3 = N1;
    a.scaled_table = false;
    a.src = 0;
    a.dst = 0;
    wm_pass_plan b;  // M1-point DFTs over a, lines (o=c, i=j1); twiddle root^(j1*(c + M2*d))
    b.column = true;
    b.logL = logM1;
    b.G = choose_G(logM1, N1);
    b.lines_inner = N1;
    b.lines_outer = M2;
    b.RO = N1 * M1;
    b.RT = N1;
    b.WO = N1;
    b.WK = N1 * M2;
    b.SH = 0;
    b.C1 = 1;
    b.C2 = M2;
    b.C3 = 1;
    b.scaled_table = true;
    b.src = 2;  // reads `out` (written by pass a)
    b.dst = 1;
    wm_pass_plan cc;  // N1-point DFTs over contiguous j1, transposing store
    cc.column = false;
    cc.logL = logN1;
    cc.G = choose_G(logN1, 1 << 20);
    cc.lines_inner = N2;
    cc.WO = 1;
    cc.WK = N2;
    cc.src = 1;
    cc.dst = 0;
    pl->passes.push_back(a);
    pl->passes.push_back(b);
    pl->passes.push_back(cc);
  }
  pl->passes.back().canonical_out = true;
  for (const auto &ps : pl->passes) {
    if (pass_smem(K, ps) > 227 * 1024) return fail(WM_EUNSUPPORTED, "pass does not fit in shared memory");
    // the shared-memory swizzle folds row indices below 512 (Smem<K>::swz)
    const bool swizzled = (K % 4 == 0) && ((K / 4) & (K / 4 - 1)) == 0 && K / 4 <= 8;
    if (swizzled && (size_t)ps.G * ((size_t)1 << ps.logL) * K * 4 > 512 * 128)
      return fail(WM_EUNSUPPORTED, "pass tile above 64 KB");
  }
  return WM_OK;
}

}  // namespace wm

using namespace wm;

extern "C" {

int wm_ntt_plan_create(const wm_field *f, int64_t n, const uint32_t *root_host, const uint32_t *root_inv_host,
                       const uint32_t *n_inv_host, wm_ntt_plan **out) {
  if (!out) return fail(WM_EINVAL, "null output pointer");
  *out = nullptr;
  if (!f) return fail(WM_EINVAL, "null field");
  if (!root_host || !root_inv_host || !n_inv_host) return fail(WM_EINVAL, "null root/root_inv/n_inv");
  if (n < 2 || (n & (n - 1))) return fail(WM_EINVAL, "transform length must be a power of two >= 2");
  if (n > ((int64_t)1 << 30)) return fail(WM_EUNSUPPORTED, "transform length above 2^30");
  const int K = f->K;
  if (!ntt_supports(K)) return fail(WM_EUNSUPPORTED, "limb count not built into the NTT kernels");
  if (f->mont && !mont_supports(K))
    return fail(WM_EUNSUPPORTED, "limb count not built into the full-width NTT kernels");
  // Shoup needs p < 2^(32K-2): guaranteed by the field's p < 2^(32K-4).
  wm_ntt_plan *pl = new wm_ntt_plan();
  pl->field = f;
  pl->K = K;
  pl->n = n;
  pl->logn = 63 - __builtin_clzll((unsigned long long)n);
  Big root(root_host, root_host + K), root_inv(root_inv_host, root_inv_host + K);
  pl->ninv = Big(n_inv_host, n_inv_host + K);
  if (f->mont) pl->ninv_mont = to_mont(pl->ninv, f->q);
  // arithmetic mode: full-width fields with two bits of headroom take the
  // Shoup / [0, 4p) path, the rest the Montgomery path (Arith<K, MODE>)
  pl->mode = ntt_mode_for(f);
  // Shoup companion of n^-1 and np = 2^(32K) - p on the host.
  {
    Big num = big_shl(pl->ninv, 32 * K, 2 * K);
    // floor(num / p) via long division over 64K bits
    Big rem(K + 1, 0u), dd = big_resize(f->q, K + 1), quo(K, 0u);
    for (int bit = 64 * K - 1; bit >= 0; --bit) {
      uint32_t carry = (num[bit / 32] >> (bit % 32)) & 1u;
      for (int j = 0; j < K + 1; ++j) {
        uint32_t nc = rem[j] >> 31;
        rem[j] = (rem[j] << 1) | carry;
        carry = nc;
      }
      if (big_ge(rem, dd)) {
        big_sub_inplace(rem, dd);
        if (bit / 32 < K) quo[bit / 32] |= 1u << (bit % 32);
      }
    }
    pl->ninv_sh = quo;
    pl->np = Big(K, 0u);
    big_sub_inplace(pl->np, f->q);
    pl->p2 = big_shl(f->q, 1, K);
    pl->p4 = big_shl(f->q, 2, K);
    pl->p3 = pl->p4;
    big_sub_inplace(pl->p3, f->q);
  }
  int rc = plan_passes(pl);
  if (rc) {
    delete pl;
    return rc;
  }
  switch (K) {
#define WM_CASE(k)                                  \
  case k:                                           \
    rc = create_tables<k>(pl, root, root_inv);      \
    break;
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      rc = fail(WM_EUNSUPPORTED, "limb count not built into the NTT kernels");
  }
  if (rc) {
    wm_ntt_plan_destroy(pl);
    return rc;
  }
  *out = pl;
  return WM_OK;
}

int wm_ntt_plan_destroy(wm_ntt_plan *p) {
  if (!p) return WM_OK;
  // the tables come from the stream-ordered allocator (plan creation must not
  // serialise other streams); destruction keeps cudaFree's semantics: wait
  // for every user on the device, then return them to the pool
  if (p->tw_fwd || p->tw_inv || p->tw_inv_scaled || p->tw_img) cudaDeviceSynchronize();
  for (uint32_t *t : {p->tw_fwd, p->tw_inv, p->tw_inv_scaled, p->tw_img})
    if (t) cudaFreeAsync(t, cudaStreamLegacy);
  if (p->tw_fwd || p->tw_inv || p->tw_inv_scaled || p->tw_img) cudaStreamSynchronize(cudaStreamLegacy);
  if (p->ws) cudaFree(p->ws);
  if (p->ws_ev) cudaEventDestroy(p->ws_ev);
  p->host.release();
  delete p;
  return WM_OK;
}

int wm_ntt_plan_info(const wm_ntt_plan *p, int *passes, int *log_sizes, int cap) {
  if (!p) return fail(WM_EINVAL, "null plan");
  if (passes) *passes = (int)p->passes.size();
  for (int i = 0; i < (int)p->passes.size() && i < cap; ++i) log_sizes[i] = p->passes[i].logL;
  return WM_OK;
}

int64_t wm_ntt_workspace_bytes(const wm_ntt_plan *p, int64_t batch) {
  if (!p || batch < 0) return -1;
  if (p->passes.size() <= 1) return 0;
  return batch * p->n * p->K * (int64_t)sizeof(uint32_t);
}

}  // extern "C"

namespace wm {
int ntt_run_internal(const wm_ntt_plan *pc, bool inverse, const uint32_t *in, uint32_t *out, int64_t batch,
                     void *workspace, cudaStream_t stream, const uint32_t *mul_by) {
  if (!pc) return fail(WM_EINVAL, "null plan");
  if (batch < 0) return fail(WM_EINVAL, "negative batch");
  if (batch == 0) return WM_OK;
  if (!in || !out) return fail(WM_EINVAL, "null data pointer");
  wm_ntt_plan *p = const_cast<wm_ntt_plan *>(pc);
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t need = wm_ntt_workspace_bytes(p, batch);
  uint32_t *ws = static_cast<uint32_t *>(workspace);
  auto run = [&](uint32_t *w) -> int {
    switch (p->K) {
#define WM_CASE(k) \
  case k:          \
    return run_passes<k>(p, inverse, in, out, batch, w, st, -1, mul_by);
      WM_NTT_KS(WM_CASE)
#undef WM_CASE
      default:
        return fail(WM_EUNSUPPORTED, "limb count not built into the NTT kernels");
    }
  };
  if (need == 0 || ws) return run(ws);
  // The plan's own workspace is shared by every caller of the plan, on any
  // stream: its uses are stream-ordered through ws_ev (each use waits for the
  // previous one, on whatever stream that ran), and it only grows once the
  // last use has completed.
  std::lock_guard<std::mutex> lk(p->ws_mu);
  if (!p->ws_ev) WM_CUDA_TRY(cudaEventCreateWithFlags(&p->ws_ev, cudaEventDisableTiming));
  if (p->ws_bytes < need) {
    if (p->ws) {
      WM_CUDA_TRY(cudaEventSynchronize(p->ws_ev));
      WM_CUDA_TRY(cudaFree(p->ws));
      p->ws = nullptr;
      p->ws_bytes = 0;
    }
    WM_CUDA_TRY(cudaMalloc(&p->ws, need));
    p->ws_bytes = need;
  }
  WM_CUDA_TRY(cudaStreamWaitEvent(st, p->ws_ev, 0));
  const int rc = run(static_cast<uint32_t *>(p->ws));
  WM_CUDA_TRY(cudaEventRecord(p->ws_ev, st));
  return rc;
}
}  // namespace wm

extern "C" {

static int ntt_run(const wm_ntt_plan *pc, bool inverse, const uint32_t *in, uint32_t *out, int64_t batch,
                   void *workspace, void *stream) {
  return wm::ntt_run_internal(pc, inverse, in, out, batch, workspace, (cudaStream_t)stream);
}

int wm_ntt_forward(const wm_ntt_plan *p, const uint32_t *in, uint32_t *out, int64_t batch, void *workspace,
                   void *stream) {
  return ntt_run(p, false, in, out, batch, workspace, stream);
}

int wm_ntt_inverse(const wm_ntt_plan *p, const uint32_t *in, uint32_t *out, int64_t batch, void *workspace,
                   void *stream) {
  return ntt_run(p, true, in, out, batch, workspace, stream);
}

int wm_ntt_convolve(const wm_ntt_plan *p, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t batch,
                    void *workspace, void *stream) {
  if (!p) return fail(WM_EINVAL, "null plan");
  if (!a || !b || !out) return fail(WM_EINVAL, "null data pointer");
  if (b == out && a != out) return fail(WM_EINVAL, "b may not alias out (out holds NTT(a) while b is read)");
  if (b == out) return fail(WM_EINVAL, "a and b may not both alias out");
  if (batch < 0) return fail(WM_EINVAL, "negative batch");
  if (batch == 0) return WM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // NTT(a) is the multiplier the last pass of NTT(b) reads.  One- and
  // two-pass plans write `out` only in their last pass, so NTT(a) can wait
  // there; a three-pass plan's first pass also writes `out`, so NTT(a) is
  // held in a stream-ordered temporary instead.
  uint32_t *hold = out;
  if (p->passes.size() > 2) {
    void *h = nullptr;
    WM_CUDA_TRY(cudaMallocAsync(&h, (size_t)batch * p->n * p->K * sizeof(uint32_t), st));
    hold = static_cast<uint32_t *>(h);
  }
  int rc = ntt_run_internal(p, false, a, hold, batch, workspace, st, nullptr);  // hold = NTT(a)
  if (!rc) rc = ntt_run_internal(p, false, b, out, batch, workspace, st, hold);  // out = NTT(b) * NTT(a), fused
  if (hold != out) {
    const cudaError_t e = cudaFreeAsync(hold, st);
    if (!rc && e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  }
  if (rc) return rc;
  return ntt_run_internal(p, true, out, out, batch, workspace, st, nullptr);  // out = INTT(...)
}

int wm_ntt_pass(const wm_ntt_plan *p, int inverse, int pass_index, const uint32_t *in, uint32_t *out,
                int64_t batch, void *stream) {
  if (!p) return fail(WM_EINVAL, "null plan");
  if (pass_index < 0 || pass_index >= (int)p->passes.size()) return fail(WM_EINVAL, "pass index out of range");
  if (batch <= 0 || !in || !out || in == out) return fail(WM_EINVAL, "bad buffers/batch");
  switch (p->K) {
#define WM_CASE(k) \
  case k:          \
    return run_passes<k>(p, inverse != 0, in, out, batch, nullptr, (cudaStream_t)stream, pass_index);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built into the NTT kernels");
  }
}

int wm_ntt_twiddles(const wm_ntt_plan *p, int inverse, int64_t count, uint32_t *out, void *stream) {
  if (!p) return fail(WM_EINVAL, "null plan");
  if (count < 0 || count > p->n) return fail(WM_EINVAL, "count out of range");
  if (count == 0) return WM_OK;
  switch (p->K) {
#define WM_CASE(k) \
  case k:          \
    return extract_twiddles<k>(p, inverse, count, out, (cudaStream_t)stream);
    WM_NTT_KS(WM_CASE)
#undef WM_CASE
    default:
      return fail(WM_EUNSUPPORTED, "limb count not built into the NTT kernels");
  }
}

}  // extern "C"
