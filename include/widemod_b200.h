/* widemod_b200 — C ABI of the B200-native multi-word modular arithmetic
 * library (vadd/vsub/vmul/axpy and radix-2 NTT/INTT over 32..1024-bit prime
 * fields).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `widemod` (reference: pkg/src/widemod/).  The reference has no compiled
 * native code: its device path is CUDA *text* produced by emit.emit_cuda
 * (emit.py:414-561) with one `extern "C" void {name}_launch(...)` symbol per
 * (kind, n, bits, word), baked constants, default stream, no error channel
 * and 32-bit `int` sizes (emit.py:456-484, 545-560; golden
 * tests/golden/mulmod_16w8.cu:126-137, tests/golden/ntt8_16w8.cu:231-240).
 * Each entry point below replaces one of those launchers (cited per function)
 * with a runtime-parameterised version that takes the modulus at run time,
 * an explicit CUDA stream, 64-bit sizes, and returns a status code.
 *
 * Conventions
 *   - Values are K x 32-bit limbs, least-significant limb first, one element
 *     after another ("element-contiguous little-endian limbs"); K = limbs of
 *     the field (wm_field_info).  A value of `bits` interface width occupies
 *     K = ceil(bits/32) limbs (no power-of-two padding, unlike the reference's
 *     WordLayout.padded_words, kernels.py:65-71).  wm_ref_to_limbs /
 *     wm_limbs_to_ref convert from/to the reference's AoS MSW-first word
 *     layout (kernels.py:418-428).
 *   - All data pointers are caller-owned DEVICE pointers unless the name says
 *     _host.  `stream` is a cudaStream_t (NULL = legacy default stream).
 *     Calls are asynchronous with respect to the host.
 *   - Inputs must be canonical residues (< modulus), as in the reference
 *     (oracle.py:7-9); outputs are canonical residues.
 *   - Every function returns WM_OK (0) or a nonzero status; wm_last_error()
 *     returns a thread-local message for the last failure on this thread.
 *   - Plans/fields are immutable after creation and may be shared between
 *     threads; calls on different streams may run concurrently.  One NTT
 *     plan's internal workspace (used when workspace == NULL) is shared by
 *     all its callers: those calls are stream-ordered one after another (each
 *     waits on the device for the previous user, on whatever stream), so pass
 *     a workspace per stream for concurrent multi-pass transforms.
 *   - Setup calls (field/plan creation) never synchronise the device or the
 *     legacy default stream: plan tables are generated on a private stream.
 */
#ifndef WIDEMOD_B200_H
#define WIDEMOD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WM_ABI_VERSION 1

#define WM_OK 0
#define WM_EINVAL 1        /* bad argument (reference: ValueError family) */
#define WM_ECUDA 2         /* CUDA runtime failure */
#define WM_EUNSUPPORTED 3  /* limb count / size not built into this library */
#define WM_ELENGTH 4       /* length mismatch (reference: LengthMismatch) */

typedef struct wm_field wm_field;
typedef struct wm_ntt_plan wm_ntt_plan;

int wm_abi_version(void);
const char *wm_last_error(void);

/* Limb count the library uses for an interface width (ceil(bits/32)), or -1
 * if that width is not built in.  Mirrors WordLayout(bits, 32).words
 * (kernels.py:61-63). */
int wm_limbs_for_bits(int bits);

/* Writes the built-in limb counts for the BLAS kernels (ntt=0) or the NTT
 * kernels (ntt=1) to out[0..cap), returns how many there are. */
int wm_supported_limbs(int ntt, int *out, int cap);

/* ---------------------------------------------------------------- fields
 * A field is a modulus q for an interface width `bits` together with the
 * device-side reduction constants.  Replaces the constants the reference
 * bakes into generated code (kernels._param_vars kernels.py:168-181,
 * oracle.compute_barrett oracle.py:109-134).  Requires
 * 2^(bits-5) < q < 2^(bits-4) (the reference's Barrett range, oracle.py:124-128)
 * or more generally 1 < q < 2^(32K-4) with bit length > 32K-36.
 * q is given as q_limbs little-endian 32-bit limbs (host memory). */
int wm_field_create(int bits, const uint32_t *q_host, int q_limbs, wm_field **out);
/* flags: WM_FIELD_KARATSUBA selects one-level (recursive for >= 16 limbs)
 * Karatsuba full products in vmul/axpy — the reference's
 * make_spec(..., strategy="karatsuba") (kernels.py:104-117, rewrite.py:234-253).
 * The NTT's Shoup multiply is a truncated product and is unaffected. */
#define WM_FIELD_KARATSUBA 1
/* WM_FIELD_MONTGOMERY: a full-width field — any odd q with bit length <= bits
 * (the paper's Montgomery mode for moduli of full bit width, PAPER.md:731;
 * e.g. secp256k1's p or BLS12-381's r at 256 bits).  Sums carry-aware,
 * products by Montgomery multiplication (vmul: two Montgomery products, axpy:
 * one with the scalar in Montgomery form); inputs and outputs stay canonical
 * residues.  Kernels for 1, 2, 4, 8, 12, 16, 24 and 32 limbs; other widths run
 * zero-padded to the next of those (wm_field_info reports the storage limbs).
 * A width whose limb count has no Barrett kernels either (513-736, 769-992
 * bits) is created as such a padded Montgomery field when q is odd. */
#define WM_FIELD_MONTGOMERY 2
/* WM_FIELD_BARRETT: always reduce products by the generic Barrett quotient
 * estimate (the reference's lower_modmul_barrett, rewrite.py:333-351).
 * Without it, a reference-range modulus of special form q = 2^m - c with
 * c < 2^32 (every modulus find_ntt_params returns, oracle.py:186-239: the
 * largest primes below 2^(bits-4)) at 72 <= m and 4 <= 32K - m <= 31 is
 * reduced by two folds t = H 2^m + L -> L + H c (K + 2 word products per
 * product instead of ~1.5 K^2), in vmul/axpy and in the NTT butterflies.
 * Results are the same canonical residues either way. */
#define WM_FIELD_BARRETT 4
int wm_field_create_ex(int bits, const uint32_t *q_host, int q_limbs, int flags, wm_field **out);
/* The reduction a field's products use: one of WM_REDUCTION_* (or a negative
 * status on error). */
#define WM_REDUCTION_BARRETT 0
#define WM_REDUCTION_MONTGOMERY 1
#define WM_REDUCTION_SPECIAL_FORM 2
int wm_field_reduction(const wm_field *f);
int wm_field_destroy(wm_field *f);
int wm_field_info(const wm_field *f, int *bits, int *limbs, int *norm_shift);

/* ---------------------------------------------------------------- BLAS
 * Replace `{kind}{n}_{bits}w{word}_launch(const w *a, const w *b, w *out,
 * int n_elems)` (emit.py:456-484) for kind in vadd/vsub/vmul: out[i] =
 * a[i] (+,-,*) b[i] mod q for i < n.  out may alias a or b.
 * Semantics: reference build_vector kernels.py:215-256. */
/* Replaces the reference's bare widening multiply `widemul_{bits}w{word}`
 * (build_wide_mul kernels.py:314-329): out[i] = a[i] * b[i] as the full
 * product, 2L limbs per element, where L = wm_limbs_for_bits(bits) is the
 * storage limb count of a and b.  No modulus; karatsuba != 0 selects the
 * Karatsuba full product (make_spec(..., strategy="karatsuba")). */
int wm_widemul(int bits, int karatsuba, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t n,
               void *stream);
int wm_vadd(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out,
            int64_t n, void *stream);
int wm_vsub(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out,
            int64_t n, void *stream);
int wm_vmul(const wm_field *f, const uint32_t *a, const uint32_t *b, uint32_t *out,
            int64_t n, void *stream);
/* Replaces the axpy launcher `(const w *a, const w *x, const w *y, w *out,
 * int n_elems)` whose scalar `a` is an un-indexed device pointer
 * (emit.py:463-472, vector_args=[False,True,True] kernels.py:228-230):
 * out[i] = a*x[i] + y[i] mod q.  Here the scalar is passed by value from
 * HOST memory (K limbs), so no device round trip is needed. */
int wm_axpy(const wm_field *f, const uint32_t *a_host, const uint32_t *x, const uint32_t *y,
            uint32_t *out, int64_t n, void *stream);

/* ---------------------------------------------------------------- NTT
 * A plan for length-n (power of two, 2 <= n <= 2^30) cyclic transforms over
 * the field's prime p = q with root of exact order n (reference NttParams,
 * oracle.py:74-82; find_ntt_params oracle.py:186-239).  root, root_inv and
 * n_inv are canonical residues, K limbs each (host memory).  Twiddle tables
 * are generated on the device at plan creation. */
int wm_ntt_plan_create(const wm_field *f, int64_t n, const uint32_t *root_host,
                       const uint32_t *root_inv_host, const uint32_t *n_inv_host,
                       wm_ntt_plan **out);
int wm_ntt_plan_destroy(wm_ntt_plan *p);
/* Number of passes and per-pass sub-transform sizes (log2) of the plan. */
int wm_ntt_plan_info(const wm_ntt_plan *p, int *passes, int *log_sizes, int cap);

/* Bytes of device workspace a call with this batch needs (0 for one-pass
 * plans).  Pass workspace=NULL to let the plan use (and grow) its own. */
int64_t wm_ntt_workspace_bytes(const wm_ntt_plan *p, int64_t batch);

/* Replace `ntt{n}_{bits}w{word}_launch(const w *in, w *x, int batch)` and the
 * intt equivalent (emit.py:545-560): for each of `batch` contiguous
 * transforms, out = NTT(in) with y[k] = sum_j x[j] root^(jk) mod p (forward)
 * or out = n^-1 sum_j x[j] root^(-jk) (inverse), natural order in and out —
 * bit-identical to reference run_ntt (kernels.py:483-499) and ntt_reference
 * (oracle.py:262-282).  in may equal out. */
int wm_ntt_forward(const wm_ntt_plan *p, const uint32_t *in, uint32_t *out, int64_t batch,
                   void *workspace, void *stream);
int wm_ntt_inverse(const wm_ntt_plan *p, const uint32_t *in, uint32_t *out, int64_t batch,
                   void *workspace, void *stream);

/* Cyclic convolution of each pair of length-n vectors (batch of them):
 * out = INTT(NTT(a) * NTT(b)) — the reference's own convolution check
 * (verify.py:195-223: run_ntt, run_vector(vmul), run_ntt(intt)) as three
 * launch sequences, with the pointwise product fused into the epilogue of
 * the forward transform of b.  a may alias out; b may not.  Three-pass plans
 * hold NTT(a) in a stream-ordered temporary (cudaMallocAsync) of
 * batch * n * K words. */
int wm_ntt_convolve(const wm_ntt_plan *p, const uint32_t *a, const uint32_t *b, uint32_t *out, int64_t batch,
                    void *workspace, void *stream);

/* Diagnostic: launch pass `pass_index` of the forward/inverse transform
 * alone, from `in` to `out` (distinct buffers), e.g. to time one kernel with
 * events.  Intermediate passes leave values in [0, 4p); only the full
 * wm_ntt_forward/inverse sequence is the transform. */
int wm_ntt_pass(const wm_ntt_plan *p, int inverse, int pass_index, const uint32_t *in, uint32_t *out,
                int64_t batch, void *stream);

/* Copies twiddle powers root^e (inverse: root_inv^e) for e in [0, count) into
 * out (device, count*K limbs): the reference twiddle_table (kernels.py:259-267)
 * is the first n/2 of them. */
int wm_ntt_twiddles(const wm_ntt_plan *p, int inverse, int64_t count, uint32_t *out,
                    void *stream);

/* ---------------------------------------------------------------- host pipeline
 * End-to-end transforms on HOST buffers in the reference layout (AoS,
 * `ref_words` words of `word_bits` bits per element, MSW first): the call a
 * reference user makes with data in host memory.  The batch is processed in
 * chunks of `chunk` transforms through a three-stage pipeline on the plan's
 * internal streams — H2D copy, {layout convert, transform(s), layout convert},
 * D2H copy — so PCIe traffic in both directions overlaps the kernels.  Host
 * buffers should be pinned (cudaHostAlloc / cudaHostRegister) for overlap.
 * mode: WM_NTT_FWD, WM_NTT_INV, or WM_NTT_FWD_INV (forward then inverse, the
 * benchmark's round trip); WM_NTT_COPY runs the same pipeline with the layout
 * conversions but no transform (the PCIe floor of the path, for measurement).  Ordered after prior work on `stream`; `stream`
 * waits for the whole pipeline, so event timing on it brackets everything. */
#define WM_NTT_FWD 0
#define WM_NTT_INV 1
#define WM_NTT_FWD_INV 2
#define WM_NTT_COPY 3
int wm_ntt_host(const wm_ntt_plan *p, int mode, int word_bits, int ref_words, const void *host_in,
                void *host_out, int64_t batch, int64_t chunk, void *stream);

/* BLAS on HOST buffers in the reference layout (`ref_words` words of
 * `word_bits` bits per element, MSW first; kernels.to_words
 * kernels.py:418-428): the end-to-end run_vector a reference user makes with
 * data in host memory (kernels.py:467-480).  op: WM_OP_VADD/VSUB/VMUL/AXPY;
 * for AXPY a_host is x, b_host is y and scalar_host the scalar (K limbs,
 * host memory), else scalar_host is ignored.  Chunks of `chunk` elements
 * (0 = auto) flow through an H2D / {convert, op, convert} / D2H pipeline on
 * the field's internal streams.  out_host may equal a_host or b_host.
 * Ordered after prior work on `stream`, which waits for the whole pipeline. */
#define WM_OP_VADD 0
#define WM_OP_VSUB 1
#define WM_OP_VMUL 2
#define WM_OP_AXPY 3
int wm_blas_host(const wm_field *f, int op, const uint32_t *scalar_host, int word_bits, int ref_words,
                 const void *a_host, const void *b_host, void *out_host, int64_t n, int64_t chunk, void *stream);

/* ---------------------------------------------------------------- distributed four-step
 * Pieces of the multi-GPU four-step NTT (one all-to-all per transform; the
 * reference has no multi-GPU path).  See paper_2501_07535_b200/dist.py.
 *   wm_transpose:        out[b][c][r] = in[b][r][c] for elements of `words` uint32s.
 *   wm_scale_transpose:  out[c][r] = in[r][c] * table[r][c] mod p (canonical),
 *                        table entries = (w, w') Shoup pairs of 2K words.
 *   wm_twiddle_table_2d: table[r][c] = root^((row0 + r) * c mod n) as Shoup pairs. */
int wm_transpose(int words, const uint32_t *in, uint32_t *out, int64_t rows, int64_t cols,
                 int64_t batch, void *stream);
int wm_scale_transpose(const wm_field *f, const uint32_t *in, const uint32_t *table, uint32_t *out,
                       int64_t rows, int64_t cols, void *stream);

/* wm_scale_transpose with the all-to-all fused in: output row c is stored into
 * dst_ptrs[c / (cols/P)] at [src_rank][c mod (cols/P)][0..rows) of that rank's
 * receive buffer ([P][cols/P][rows] elements).  dst_ptrs (host array of P
 * device addresses, P <= 16) are peer-mapped buffers (symmetric memory over
 * NVLink) or local buffers.  Replaces the exchange step the reference does not
 * have. */
int wm_scale_transpose_scatter(const wm_field *f, const uint32_t *in, const uint32_t *table,
                               const uint64_t *dst_ptrs, int P, int src_rank, int64_t rows, int64_t cols,
                               void *stream);
int wm_twiddle_table_2d(const wm_field *f, int64_t n, const uint32_t *root_host, int64_t row0,
                        int64_t rows, int64_t cols, uint32_t *table, void *stream);

/* Factored twiddles for the four-step: root^e = hi[e >> logB] * lo[e mod 2^logB]
 * (e < n), two tables of 2^logB and n / 2^logB entries of K words (in the
 * field's product form: Montgomery form for full-width fields) — O(sqrt n)
 * memory instead of wm_twiddle_table_2d's rows x cols Shoup pairs.
 *   wm_twiddle_factors:    fill lo[0 .. 2^logB) and hi[0 .. n/2^logB).
 *   wm_scale_transpose_fx: out[c][r] = in[r][c] * root^((row0 + r) c mod n)
 *     (canonical).  P == 0: into `out` ([cols][rows]).  P >= 1: output row
 *     c goes to dst_ptrs[c / (cols/P)] — layout 0 at [src_rank][c mod cols/P]
 *     [rows] (an all-to-all's block layout), layout 1 at [c mod cols/P]
 *     [src_rank * rows + r] (the receiving rank's phase-2 rows: no block
 *     transpose needed). */
int wm_twiddle_factors(const wm_field *f, int64_t n, const uint32_t *root_host, int logB, uint32_t *lo,
                       uint32_t *hi, void *stream);
int wm_scale_transpose_fx(const wm_field *f, const uint32_t *in, const uint32_t *lo, const uint32_t *hi, int logB,
                          int64_t n, int64_t row0, uint32_t *out, const uint64_t *dst_ptrs, int P, int src_rank,
                          int layout, int64_t rows, int64_t cols, void *stream);

/* ---------------------------------------------------------------- diagnostics
 * Roofline inputs for the integer-bound kernels (bench.py).
 *   wm_probe_imad_wide: launch a kernel of 8 independent 32x32->64 product
 *     chains per thread at full occupancy (mode 0: mad.wide.u32 with a 64-bit
 *     addend, mode 1: mul.wide.u32), `iters` steps each; *products = word
 *     products it executes.  Time it with events on `stream` for this GPU's
 *     product throughput.  sink: 8 bytes of device scratch.
 *   wm_ntt_pass_work: field multiplications the pass kernel `pass_index` of a
 *     forward (inverse != 0: inverse) transform executes for `batch`
 *     transforms, and the word products they cost in the plan's arithmetic
 *     (32x32->32 low products count one half).
 *   wm_blas_work: the same per element of a BLAS op. */
int wm_probe_imad_wide(int mode, int64_t iters, uint64_t *sink, void *stream, int64_t *products);
int wm_ntt_pass_work(const wm_ntt_plan *p, int inverse, int pass_index, int64_t batch, int64_t *field_muls,
                     double *word_products);
/* Word products one element of `op` (WM_OP_*) executes in the field's
 * arithmetic (mirrors the BLAS templates: Karatsuba levels, truncated Barrett
 * quotient, or the special-form folds; a 32x32->32 low product counts one
 * half; 0 for vadd/vsub).  WM_EUNSUPPORTED for Montgomery fields. */
int wm_blas_work(const wm_field *f, int op, double *word_products);

/* ---------------------------------------------------------------- layout
 * Reference layout: AoS, `ref_words` words of `word_bits` (32 or 64) per
 * element, most-significant word first (kernels.to_words kernels.py:418-421;
 * emit_cuda element pointers `a + i * per_arg`, emit.py:466-470).  Words above
 * the K limbs must be zero on input and are written as zero on output. */
int wm_ref_to_limbs(int word_bits, int ref_words, int limbs, const void *ref, uint32_t *out,
                    int64_t n, void *stream);
int wm_limbs_to_ref(int word_bits, int ref_words, int limbs, const uint32_t *in, void *ref,
                    int64_t n, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* WIDEMOD_B200_H */
