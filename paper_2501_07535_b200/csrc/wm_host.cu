// Host-buffer pipelines (wm_ntt_host, wm_blas_host): the end-to-end path a
// reference user takes — data in host memory in the reference's AoS
// MSW-first word layout (kernels.to_words, kernels.py:418-428) — with PCIe
// traffic overlapped against the kernels ("the host
// boundary's throughput").
//
// Owner-held streams (HostPipe) form a pipeline over chunks with kSlots
// staging slots in device memory:
//   h2d stream:      wait slot free -> memcpy the chunk's inputs -> record ev_in
//   compute streams: wait ev_in -> ref->limbs, kernels, limbs->ref,
//                    memcpy to host_out -> record ev_out (slot free)
// (WM_HOST_POST=0: the D2H copies on a dedicated stream after ev_comp).
// PCIe is full duplex, so H2D and D2H of different chunks run at once.  A
// small chunk's kernels fill only part of the GPU (a 2^16-point, 256-bit
// chunk of 2 transforms is 64 CTAs per pass), so chunks round-robin over
// kComp compute streams and the kernels of consecutive chunks run
// concurrently; the copies, not the kernels, then bound the pipeline.
#include <algorithm>
#include <cstdlib>
#include <functional>
#include <vector>

#include "wm_internal.cuh"

namespace wm {

int HostPipe::ensure(int64_t bytes) {
  if (!ready) {
    for (int i = 0; i < kStreams; ++i) WM_CUDA_TRY(cudaStreamCreateWithFlags(&hs[i], cudaStreamNonBlocking));
    for (int s = 0; s < kSlots; ++s) {
      WM_CUDA_TRY(cudaEventCreateWithFlags(&ev_in[s], cudaEventDisableTiming));
      WM_CUDA_TRY(cudaEventCreateWithFlags(&ev_comp[s], cudaEventDisableTiming));
      WM_CUDA_TRY(cudaEventCreateWithFlags(&ev_out[s], cudaEventDisableTiming));
    }
    WM_CUDA_TRY(cudaEventCreateWithFlags(&ev_entry, cudaEventDisableTiming));
    WM_CUDA_TRY(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    ready = true;
  }
  if (slot_bytes < bytes) {
    for (int i = 0; i < kStreams; ++i) WM_CUDA_TRY(cudaStreamSynchronize(hs[i]));
    for (int s = 0; s < kSlots; ++s) {
      if (slot_mem[s]) WM_CUDA_TRY(cudaFree(slot_mem[s]));
      slot_mem[s] = nullptr;
    }
    slot_bytes = 0;
    for (int s = 0; s < kSlots; ++s) WM_CUDA_TRY(cudaMalloc(&slot_mem[s], bytes));
    slot_bytes = bytes;
  }
  return WM_OK;
}

void HostPipe::release() {
  if (!ready) return;
  for (int i = 0; i < kStreams; ++i) {
    cudaStreamSynchronize(hs[i]);
    cudaStreamDestroy(hs[i]);
  }
  for (int s = 0; s < kSlots; ++s) {
    cudaEventDestroy(ev_in[s]);
    cudaEventDestroy(ev_comp[s]);
    cudaEventDestroy(ev_out[s]);
    if (slot_mem[s]) cudaFree(slot_mem[s]);
    slot_mem[s] = nullptr;
  }
  cudaEventDestroy(ev_entry);
  cudaEventDestroy(ev_done);
  slot_bytes = 0;
  ready = false;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Chunk sizes over `total` units: an explicit chunk as given; auto
// (chunk == 0, `target` units per chunk) ramps up from small chunks and back
// down at the end so the pipeline's fill (first H2D alone) and drain (last
// kernels + D2H alone) cost a fraction of a full chunk.
static std::vector<int64_t> chunk_schedule(int64_t total, int64_t chunk, int64_t target, int64_t ramp_from) {
  std::vector<int64_t> sizes;
  if (chunk == 0) {
    chunk = std::min<int64_t>(total, std::max<int64_t>(1, target));
    std::vector<int64_t> ramp;
    for (int64_t r = std::max<int64_t>(1, ramp_from); r < chunk; r *= 2) ramp.push_back(r);
    int64_t ramp_total = 0;
    for (int64_t r : ramp) ramp_total += 2 * r;
    if (total >= ramp_total + chunk) {
      int64_t mid = total - ramp_total;
      sizes = ramp;
      for (; mid > 0; mid -= chunk) sizes.push_back(std::min(chunk, mid));
      for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) sizes.push_back(*it);
      return sizes;
    }
  }
  chunk = std::min(chunk, total);
  for (int64_t t = 0; t < total; t += chunk) sizes.push_back(std::min(chunk, total - t));
  return sizes;
}

// One pipelined pass over `sizes` chunks.  Inputs: nin host arrays of
// in_unit bytes per unit, staged into the slot's first nin regions; the
// compute callback (chunk units, device inputs, scratch, stream) returns the
// device pointer holding the chunk's output (out_unit bytes per unit), which
// is copied back to host_out.  Slot layout: [in 0][in 1]..[scratch].
using ChunkFn = std::function<int(int64_t nt, void *const *d_in, char *scratch, cudaStream_t st, void **d_out)>;

static int run_pipeline(HostPipe &hp, const std::vector<int64_t> &sizes, int nin, const void *const *host_in,
                        size_t in_unit, void *host_out, size_t out_unit, size_t scratch_bytes, const ChunkFn &fn,
                        cudaStream_t user) {
  int64_t max_chunk = 0;
  for (int64_t c : sizes) max_chunk = std::max(max_chunk, c);
  const size_t in_sz = align256(in_unit * (size_t)max_chunk);
  const size_t slot = nin * in_sz + align256(scratch_bytes);
  std::lock_guard<std::mutex> lk(hp.mu);
  int rc = hp.ensure((int64_t)slot);
  if (rc) return rc;
  cudaStream_t h2d = hp.hs[0], d2h = hp.hs[1];
  // A/B knobs, read per call so one process can interleave settings
  const char *e_ahead = getenv("WM_HOST_AHEAD");
  const int ahead = std::min(std::max(e_ahead ? atoi(e_ahead) : HostPipe::kSlots, 1), HostPipe::kSlots);
  // Each chunk's D2H is issued on its compute stream right after its kernels
  // (one cross-stream hop per chunk instead of two): 256-bit 2^16 x 64
  // forward+inverse 3.24 -> 3.06 ms per call against a 2.68 ms copy floor
  // (profiles/r02_e2e_ab_post.txt).  WM_HOST_POST=0 restores the dedicated
  // D2H stream (A/B).
  const char *e_post = getenv("WM_HOST_POST");
  const bool post = !e_post || atoi(e_post) != 0;
  WM_CUDA_TRY(cudaEventRecord(hp.ev_entry, user));
  for (int i = 0; i < HostPipe::kStreams; ++i) WM_CUDA_TRY(cudaStreamWaitEvent(hp.hs[i], hp.ev_entry, 0));
  int64_t u0 = 0;
  for (size_t c = 0; c < sizes.size(); ++c) {
    const int s = (int)(c % HostPipe::kSlots);
    cudaStream_t comp = hp.hs[2 + c % HostPipe::kComp];
    const int64_t nt = sizes[c];
    char *base = static_cast<char *>(hp.slot_mem[s]);
    void *d_in[4];
    // H2D may run `ahead` chunks in front of the D2H stream (slot reuse needs
    // ahead <= kSlots); a shorter lead keeps both copy directions busy together
    if (c >= (size_t)ahead) WM_CUDA_TRY(cudaStreamWaitEvent(h2d, hp.ev_out[(c - ahead) % HostPipe::kSlots], 0));
    for (int k = 0; k < nin; ++k) {
      d_in[k] = base + k * in_sz;
      WM_CUDA_TRY(cudaMemcpyAsync(d_in[k], static_cast<const char *>(host_in[k]) + in_unit * u0, in_unit * nt,
                                  cudaMemcpyHostToDevice, h2d));
    }
    WM_CUDA_TRY(cudaEventRecord(hp.ev_in[s], h2d));
    WM_CUDA_TRY(cudaStreamWaitEvent(comp, hp.ev_in[s], 0));
    void *d_out = nullptr;
    rc = fn(nt, d_in, base + nin * in_sz, comp, &d_out);
    if (rc) return rc;
    if (post) {  // the chunk's D2H follows its kernels on the same stream (one hop fewer)
      WM_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(host_out) + out_unit * u0, d_out, out_unit * nt,
                                  cudaMemcpyDeviceToHost, comp));
      WM_CUDA_TRY(cudaEventRecord(hp.ev_out[s], comp));
    } else {
      WM_CUDA_TRY(cudaEventRecord(hp.ev_comp[s], comp));
      WM_CUDA_TRY(cudaStreamWaitEvent(d2h, hp.ev_comp[s], 0));
      WM_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(host_out) + out_unit * u0, d_out, out_unit * nt,
                                  cudaMemcpyDeviceToHost, d2h));
      WM_CUDA_TRY(cudaEventRecord(hp.ev_out[s], d2h));
    }
    u0 += nt;
  }
  if (post) {  // join: the last chunk of every compute stream covers its earlier ones
    const size_t nc = sizes.size();
    for (size_t c = nc > (size_t)HostPipe::kComp ? nc - HostPipe::kComp : 0; c < nc; ++c)
      WM_CUDA_TRY(cudaStreamWaitEvent(d2h, hp.ev_out[c % HostPipe::kSlots], 0));
  }
  WM_CUDA_TRY(cudaEventRecord(hp.ev_done, d2h));
  WM_CUDA_TRY(cudaStreamWaitEvent(user, hp.ev_done, 0));
  // keep the other internal streams ordered behind the finished pipeline
  for (int i = 0; i < HostPipe::kStreams; ++i)
    if (hp.hs[i] != d2h) WM_CUDA_TRY(cudaStreamWaitEvent(hp.hs[i], hp.ev_done, 0));
  return WM_OK;
}

}  // namespace wm

using namespace wm;

extern "C" int wm_ntt_host(const wm_ntt_plan *pc, int mode, int word_bits, int ref_words, const void *host_in,
                           void *host_out, int64_t batch, int64_t chunk, void *stream) {
  if (!pc) return fail(WM_EINVAL, "null plan");
  if (mode < WM_NTT_FWD || mode > WM_NTT_COPY) return fail(WM_EINVAL, "bad mode");
  if (word_bits != 32 && word_bits != 64) return fail(WM_EINVAL, "word_bits must be 32 or 64");
  if ((int64_t)ref_words * word_bits < pc->field->bits) return fail(WM_EINVAL, "reference words too narrow");
  if (batch < 0 || chunk < 0) return fail(WM_EINVAL, "negative batch/chunk");
  if (batch == 0) return WM_OK;
  if (!host_in || !host_out) return fail(WM_EINVAL, "null host pointer");
  wm_ntt_plan *p = const_cast<wm_ntt_plan *>(pc);
  const int64_t n = p->n;
  const int K = p->K;
  // auto chunks: ~8 MiB of limbs (PCIe runs at ~90 GB/s both ways from 4 MiB
  // chunks up, profiles/r01_pcie_chunks.txt); no ramp (with the D2H on the
  // compute streams the ramped schedule was 1.5 % slower, profiles/r02_e2e_post.txt)
  const int64_t target = std::max<int64_t>(1, (int64_t)(8 << 20) / (n * K * 4));
  const char *e_ramp = getenv("WM_HOST_RAMP");  // A/B knob: ramp the chunk sizes from this many transforms
  const int64_t ramp_from = e_ramp && atoi(e_ramp) > 0 ? atoi(e_ramp) : target;
  const std::vector<int64_t> sizes = chunk_schedule(batch, chunk, target, ramp_from);
  int64_t max_chunk = 0;
  for (int64_t c : sizes) max_chunk = std::max(max_chunk, c);
  const size_t ref_unit = (size_t)n * ref_words * (word_bits / 8);
  const size_t limb_sz = align256((size_t)n * K * 4 * max_chunk);
  const size_t ws_sz = align256((size_t)std::max<int64_t>(0, wm_ntt_workspace_bytes(p, max_chunk)));
  ChunkFn fn = [&](int64_t nt, void *const *d_in, char *scratch, cudaStream_t comp, void **d_out) -> int {
    uint32_t *d_a = reinterpret_cast<uint32_t *>(scratch);
    uint32_t *d_b = reinterpret_cast<uint32_t *>(scratch + limb_sz);
    void *d_ws = ws_sz ? scratch + 2 * limb_sz : nullptr;
    int rc = wm_ref_to_limbs(word_bits, ref_words, K, d_in[0], d_a, n * nt, comp);
    if (rc) return rc;
    uint32_t *res = d_a;
    if (mode == WM_NTT_FWD || mode == WM_NTT_FWD_INV) {
      rc = ntt_run_internal(p, false, d_a, d_b, nt, d_ws, comp);
      if (rc) return rc;
      res = d_b;
    }
    if (mode == WM_NTT_INV || mode == WM_NTT_FWD_INV) {
      uint32_t *dst = (res == d_a) ? d_b : d_a;
      rc = ntt_run_internal(p, true, res, dst, nt, d_ws, comp);
      if (rc) return rc;
      res = dst;
    }
    rc = wm_limbs_to_ref(word_bits, ref_words, K, res, d_in[0], n * nt, comp);
    *d_out = d_in[0];
    return rc;
  };
  const void *ins[1] = {host_in};
  return run_pipeline(p->host, sizes, 1, ins, ref_unit, host_out, ref_unit, 2 * limb_sz + ws_sz, fn,
                      (cudaStream_t)stream);
}

extern "C" int wm_blas_host(const wm_field *fc, int op, const uint32_t *scalar_host, int word_bits, int ref_words,
                            const void *a_host, const void *b_host, void *out_host, int64_t n, int64_t chunk,
                            void *stream) {
  if (!fc) return fail(WM_EINVAL, "null field");
  if (op < WM_OP_VADD || op > WM_OP_AXPY) return fail(WM_EINVAL, "bad op");
  if (op == WM_OP_AXPY && !scalar_host) return fail(WM_EINVAL, "axpy needs a scalar");
  if (word_bits != 32 && word_bits != 64) return fail(WM_EINVAL, "word_bits must be 32 or 64");
  if ((int64_t)ref_words * word_bits < fc->bits) return fail(WM_EINVAL, "reference words too narrow");
  if (n < 0 || chunk < 0) return fail(WM_EINVAL, "negative length/chunk");
  if (n == 0) return WM_OK;
  if (!a_host || !b_host || !out_host) return fail(WM_EINVAL, "null host pointer");
  wm_field *f = const_cast<wm_field *>(fc);
  const int K = f->K;
  // auto chunks: ~4 MiB of limbs per operand, ramping up from 1/16 of that
  const int64_t target = (int64_t)(4 << 20) / (K * 4);
  const std::vector<int64_t> sizes = chunk_schedule(n, chunk, target, target / 16);
  int64_t max_chunk = 0;
  for (int64_t c : sizes) max_chunk = std::max(max_chunk, c);
  const size_t ref_unit = (size_t)ref_words * (word_bits / 8);
  const size_t limb_sz = align256((size_t)K * 4 * max_chunk);
  ChunkFn fn = [&](int64_t nt, void *const *d_in, char *scratch, cudaStream_t comp, void **d_out) -> int {
    uint32_t *d_a = reinterpret_cast<uint32_t *>(scratch);
    uint32_t *d_b = reinterpret_cast<uint32_t *>(scratch + limb_sz);
    int rc = wm_ref_to_limbs(word_bits, ref_words, K, d_in[0], d_a, nt, comp);
    if (!rc) rc = wm_ref_to_limbs(word_bits, ref_words, K, d_in[1], d_b, nt, comp);
    if (rc) return rc;
    switch (op) {
      case WM_OP_VADD: rc = wm_vadd(f, d_a, d_b, d_a, nt, comp); break;
      case WM_OP_VSUB: rc = wm_vsub(f, d_a, d_b, d_a, nt, comp); break;
      case WM_OP_VMUL: rc = wm_vmul(f, d_a, d_b, d_a, nt, comp); break;
      default: rc = wm_axpy(f, scalar_host, d_a, d_b, d_a, nt, comp); break;
    }
    if (rc) return rc;
    rc = wm_limbs_to_ref(word_bits, ref_words, K, d_a, d_in[0], nt, comp);
    *d_out = d_in[0];
    return rc;
  };
  const void *ins[2] = {a_host, b_host};
  return run_pipeline(f->host, sizes, 2, ins, ref_unit, out_host, ref_unit, 2 * limb_sz, fn, (cudaStream_t)stream);
}
