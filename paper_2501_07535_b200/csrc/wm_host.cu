// Host-buffer pipeline (wm_ntt_host): the end-to-end path a reference user
// takes — data in host memory in the reference's AoS MSW-first word layout
// (kernels.to_words, kernels.py:418-428) — with PCIe traffic overlapped
// against the kernels ("the host boundary's
// throughput").
//
// Plan-owned streams form a pipeline over chunks of `chunk` transforms with
// kSlots staging slots in device memory:
//   h2d stream:      wait slot free -> memcpy host_in chunk -> record ev_in
//   compute streams: wait ev_in -> ref->limbs, NTT[/INTT], limbs->ref -> ev_comp
//   d2h stream:      wait ev_comp -> memcpy to host_out -> record ev_out (slot free)
// PCIe is full duplex, so H2D and D2H of different chunks run at once.  A
// small chunk's kernels fill only part of the GPU (a 2^16-point, 256-bit
// chunk of 2 transforms is 64 CTAs per pass), so chunks round-robin over
// kComp compute streams and the kernels of consecutive chunks run
// concurrently; the copies, not the kernels, then bound the pipeline.
#include <algorithm>
#include <vector>

#include "wm_internal.cuh"

namespace wm {

static int ensure_host_pipeline(wm_ntt_plan *p, int64_t slot_bytes) {
  if (!p->host_ready) {
    for (int i = 0; i < wm_ntt_plan::kStreams; ++i)
      WM_CUDA_TRY(cudaStreamCreateWithFlags(&p->hs[i], cudaStreamNonBlocking));
    for (int s = 0; s < wm_ntt_plan::kSlots; ++s) {
      WM_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_in[s], cudaEventDisableTiming));
      WM_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_comp[s], cudaEventDisableTiming));
      WM_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_out[s], cudaEventDisableTiming));
    }
    WM_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_entry, cudaEventDisableTiming));
    WM_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
    p->host_ready = true;
  }
  if (p->slot_bytes < slot_bytes) {
    for (int i = 0; i < wm_ntt_plan::kStreams; ++i) WM_CUDA_TRY(cudaStreamSynchronize(p->hs[i]));
    for (int s = 0; s < wm_ntt_plan::kSlots; ++s) {
      if (p->slot_mem[s]) WM_CUDA_TRY(cudaFree(p->slot_mem[s]));
      p->slot_mem[s] = nullptr;
    }
    p->slot_bytes = 0;
    for (int s = 0; s < wm_ntt_plan::kSlots; ++s) WM_CUDA_TRY(cudaMalloc(&p->slot_mem[s], slot_bytes));
    p->slot_bytes = slot_bytes;
  }
  return WM_OK;
}

int release_host_pipeline(wm_ntt_plan *p) {
  if (!p->host_ready) return WM_OK;
  for (int i = 0; i < wm_ntt_plan::kStreams; ++i) {
    cudaStreamSynchronize(p->hs[i]);
    cudaStreamDestroy(p->hs[i]);
  }
  for (int s = 0; s < wm_ntt_plan::kSlots; ++s) {
    cudaEventDestroy(p->ev_in[s]);
    cudaEventDestroy(p->ev_comp[s]);
    cudaEventDestroy(p->ev_out[s]);
    if (p->slot_mem[s]) cudaFree(p->slot_mem[s]);
  }
  cudaEventDestroy(p->ev_entry);
  cudaEventDestroy(p->ev_done);
  p->host_ready = false;
  return WM_OK;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

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
  // Chunk schedule.  auto (chunk == 0): ~8 MiB of limbs per chunk (PCIe runs
  // at ~90 GB/s both ways from 4 MiB chunks up, profiles/r01_pcie_chunks.txt),
  // with the chunks at both ends halved down to one transform so the
  // pipeline's fill (first H2D alone) and drain (last kernels + D2H alone)
  // cost a fraction of a full chunk.  An explicit chunk size is used as given.
  std::vector<int64_t> sizes;
  if (chunk == 0) {
    chunk = std::min<int64_t>(batch, std::max<int64_t>(1, (int64_t)(8 << 20) / (n * K * 4)));
    std::vector<int64_t> ramp;
    for (int64_t r = 1; r < chunk; r *= 2) ramp.push_back(r);
    int64_t ramp_total = 0;
    for (int64_t r : ramp) ramp_total += 2 * r;
    if (batch >= ramp_total + chunk) {
      int64_t mid = batch - ramp_total;
      sizes = ramp;
      for (; mid > 0; mid -= chunk) sizes.push_back(std::min(chunk, mid));
      for (auto it = ramp.rbegin(); it != ramp.rend(); ++it) sizes.push_back(*it);
    }
  }
  chunk = std::min(chunk, batch);
  if (sizes.empty())
    for (int64_t t = 0; t < batch; t += chunk) sizes.push_back(std::min(chunk, batch - t));
  const size_t ref_bytes_per_t = (size_t)n * ref_words * (word_bits / 8);
  const size_t limb_bytes_per_t = (size_t)n * K * 4;
  const size_t ref_sz = align256(ref_bytes_per_t * chunk);
  const size_t limb_sz = align256(limb_bytes_per_t * chunk);
  const size_t ws_sz = align256((size_t)std::max<int64_t>(0, wm_ntt_workspace_bytes(p, chunk)));
  const size_t slot = ref_sz + 2 * limb_sz + ws_sz;

  std::lock_guard<std::mutex> lk(p->host_mu);
  int rc = ensure_host_pipeline(p, (int64_t)slot);
  if (rc) return rc;
  cudaStream_t user = (cudaStream_t)stream;
  cudaStream_t h2d = p->hs[0], d2h = p->hs[1];
  WM_CUDA_TRY(cudaEventRecord(p->ev_entry, user));
  for (int i = 0; i < wm_ntt_plan::kStreams; ++i) WM_CUDA_TRY(cudaStreamWaitEvent(p->hs[i], p->ev_entry, 0));

  const int64_t nchunks = (int64_t)sizes.size();
  int64_t t_next = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int s = (int)(c % wm_ntt_plan::kSlots);
    cudaStream_t comp = p->hs[2 + c % wm_ntt_plan::kComp];
    const int64_t t0 = t_next;
    const int64_t nt = sizes[c];
    t_next += nt;
    char *base = static_cast<char *>(p->slot_mem[s]);
    void *d_ref = base;
    uint32_t *d_a = reinterpret_cast<uint32_t *>(base + ref_sz);
    uint32_t *d_b = reinterpret_cast<uint32_t *>(base + ref_sz + limb_sz);
    void *d_ws = ws_sz ? base + ref_sz + 2 * limb_sz : nullptr;
    const size_t rb = ref_bytes_per_t * nt;
    if (c >= wm_ntt_plan::kSlots) WM_CUDA_TRY(cudaStreamWaitEvent(h2d, p->ev_out[s], 0));
    WM_CUDA_TRY(cudaMemcpyAsync(d_ref, static_cast<const char *>(host_in) + ref_bytes_per_t * t0, rb,
                                cudaMemcpyHostToDevice, h2d));
    WM_CUDA_TRY(cudaEventRecord(p->ev_in[s], h2d));

    WM_CUDA_TRY(cudaStreamWaitEvent(comp, p->ev_in[s], 0));
    rc = wm_ref_to_limbs(word_bits, ref_words, K, d_ref, d_a, n * nt, comp);
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
    rc = wm_limbs_to_ref(word_bits, ref_words, K, res, d_ref, n * nt, comp);
    if (rc) return rc;
    WM_CUDA_TRY(cudaEventRecord(p->ev_comp[s], comp));

    WM_CUDA_TRY(cudaStreamWaitEvent(d2h, p->ev_comp[s], 0));
    WM_CUDA_TRY(cudaMemcpyAsync(static_cast<char *>(host_out) + ref_bytes_per_t * t0, d_ref, rb,
                                cudaMemcpyDeviceToHost, d2h));
    WM_CUDA_TRY(cudaEventRecord(p->ev_out[s], d2h));
  }
  WM_CUDA_TRY(cudaEventRecord(p->ev_done, d2h));
  WM_CUDA_TRY(cudaStreamWaitEvent(user, p->ev_done, 0));
  // keep the other internal streams ordered behind the finished pipeline
  for (int i = 0; i < wm_ntt_plan::kStreams; ++i)
    if (p->hs[i] != d2h) WM_CUDA_TRY(cudaStreamWaitEvent(p->hs[i], p->ev_done, 0));
  return WM_OK;
}
