"""A CUDA backend for the reference emitter's launcher ABI.

The reference's ``emit.emit_cuda`` (emit.py:414-561) writes CUDA text whose
host entry points are ``extern "C" void {name}_launch(...)``: element kernels
``(const w *a, const w *b, [const w *q, const w *mu,] w *out, int n_elems)``
(emit.py:456-484) and transforms ``(const w *in, w *x, int batch)``
(emit.py:545-560), with the modulus, twiddles and bit-reversal table baked in.
Its transform text cannot be compiled for n >= 2^12 at 256 bits (64 KB
__constant__ limit), and at 256 bits its 1024-thread launches do not fit the
register file (bench.py reference_gpu).

``emit_cuda_launcher`` writes a translation unit that exports the *same*
symbol names and signatures, in the reference's AoS MSW-first word layout,
implemented by libwidemod_b200 (layout conversion + the sm_100a kernels): a
program built from ``widemod`` that links the emitted object keeps working at
every size.  Like the reference's output, parameters are baked into the
text (as wm_field / wm_ntt_plan created on first call).
"""

from __future__ import annotations

from .kernels import NTT_KINDS, SCALAR_KINDS, VECTOR_KINDS, DeviceKernel

_TNAME = {32: "uint32_t", 64: "uint64_t"}


def _limbs_lit(v: int, K: int) -> str:
    words = [(v >> (32 * i)) & 0xFFFFFFFF for i in range(K)]
    return "{" + ", ".join(f"0x{w:08x}u" for w in words) + "}"


def emit_cuda_launcher(program: DeviceKernel) -> str:
    """C++ source exporting the reference launcher ABI for `program`."""
    spec = program.spec
    lay = spec.layout
    word = lay.word_bits
    if word not in _TNAME:
        raise ValueError(f"the device layout converters take 32- or 64-bit words, not {word}")
    attrs = program.attributes
    name = program.name
    K = lay.limbs
    per_arg = lay.padded_words
    w = f"w{word}"
    q = program.modulus
    lines = [
        f"/* {name}: reference launcher ABI (emit.py:456-484/545-560) backed by libwidemod_b200 (sm_100a). */",
        "#include <stdint.h>",
        "#include <stddef.h>",
        "#include <stdio.h>",
        "#include <mutex>",
        "#include <cuda_runtime.h>",
        '#include "widemod_b200.h"',
        "",
        f"typedef {_TNAME[word]} {w};",
        f"static const uint32_t Q_[{K}] = {_limbs_lit(q, K)};",
        "static wm_field *field_ = NULL;",
        "static uint32_t *scratch_ = NULL;",
        "static size_t scratch_words_ = 0;",
        "static std::mutex mu_;  /* the launcher's field, plan and scratch are shared by all callers */",
        "static int status_ = WM_OK;",
        "",
        "/* The reference launchers return void (no error channel): a failure is",
        f"   reported on stderr and kept for {name}_status(). */",
        "static bool ok_(int rc, const char *what) {",
        "    if (rc == WM_OK) return true;",
        "    status_ = rc;",
        f'    fprintf(stderr, "{name}: %s failed (%d): %s\\n", what, rc, wm_last_error());',
        "    return false;",
        "}",
        "",
        f'extern "C" int {name}_status(void) {{ std::lock_guard<std::mutex> g(mu_); return status_; }}',
        "",
        "static uint32_t *scratch(size_t words) {",
        "    if (words > scratch_words_) {",
        "        if (scratch_) cudaFree(scratch_);",
        "        scratch_ = NULL;",
        "        scratch_words_ = 0;",
        "        if (cudaMalloc((void **)&scratch_, words * sizeof(uint32_t)) != cudaSuccess) {",
        "            ok_(WM_ECUDA, \"scratch cudaMalloc\");",
        "            scratch_ = NULL;",
        "            return NULL;",
        "        }",
        "        scratch_words_ = words;",
        "    }",
        "    return scratch_;",
        "}",
        "",
        "static bool init_field(void) {",
        f"    return field_ || ok_(wm_field_create({lay.bits}, Q_, {K}, &field_), \"wm_field_create\");",
        "}",
        "",
    ]
    if spec.kind in NTT_KINDS:
        nt = spec.ntt
        n = nt.n
        inverse = spec.kind == "intt"
        lines += [
            f"static const uint32_t ROOT_[{K}] = {_limbs_lit(nt.root, K)};",
            f"static const uint32_t ROOT_INV_[{K}] = {_limbs_lit(nt.root_inv, K)};",
            f"static const uint32_t N_INV_[{K}] = {_limbs_lit(nt.n_inv, K)};",
            "static wm_ntt_plan *plan_ = NULL;",
            "",
            f'extern "C" void {name}_launch(const {w} *in, {w} *x, int batch) {{',
            "    std::lock_guard<std::mutex> g(mu_);",
            "    if (batch <= 0 || !init_field()) return;",
            f"    if (!plan_ && !ok_(wm_ntt_plan_create(field_, {n}, ROOT_, ROOT_INV_, N_INV_, &plan_), "
            f"\"wm_ntt_plan_create\")) return;",
            f"    const int64_t elems = (int64_t){n} * batch;",
            f"    uint32_t *t = scratch((size_t)elems * {K});",
            "    if (!t) return;",
            f"    if (!ok_(wm_ref_to_limbs({word}, {per_arg}, {K}, in, t, elems, NULL), \"wm_ref_to_limbs\")) return;",
            f"    if (!ok_(wm_ntt_{'inverse' if inverse else 'forward'}(plan_, t, t, batch, NULL, NULL), "
            f"\"wm_ntt\")) return;",
            f"    ok_(wm_limbs_to_ref({word}, {per_arg}, {K}, t, x, elems, NULL), \"wm_limbs_to_ref\");",
            "}",
        ]
        return "\n".join(lines) + "\n"
    kind = spec.kind
    if kind in SCALAR_KINDS:
        kind = {"addmod": "vadd", "submod": "vsub", "mulmod": "vmul"}[kind]
    if kind not in VECTOR_KINDS:
        raise ValueError(f"no launcher for {spec.kind}")
    args = list(attrs["arg_names"])
    params = ", ".join(f"const {w} *{a}" for a in args) + f", {w} *out, int n_elems"
    conv = (f"    if (!ok_(wm_ref_to_limbs({word}, {per_arg}, {K}, %s, %s, n_elems, NULL), "
            f"\"wm_ref_to_limbs\")) return;")
    lines += [f'extern "C" void {name}_launch({params}) {{',
              "    std::lock_guard<std::mutex> g(mu_);",
              "    if (n_elems <= 0 || !init_field()) return;",
              f"    uint32_t *t = scratch((size_t)n_elems * {3 * K});",
              "    if (!t) return;",
              f"    uint32_t *A = t, *B = t + (size_t)n_elems * {K}, *O = t + (size_t)n_elems * {2 * K};"]
    if kind == "axpy":
        # the scalar is an un-indexed device pointer (vector_args=[False,True,True], kernels.py:228-230)
        lines += [f"    {w} s_host[{per_arg}];",
                  "    if (cudaMemcpy(s_host, a, sizeof(s_host), cudaMemcpyDeviceToHost) != cudaSuccess) {",
                  "        ok_(WM_ECUDA, \"scalar cudaMemcpy\");",
                  "        return;",
                  "    }",
                  f"    uint32_t s_limbs[{K}];",
                  f"    for (int j = 0; j < {K}; ++j) {{",
                  f"        int bit = 32 * j, wi = {per_arg} - 1 - bit / {word};",
                  f"        s_limbs[j] = (uint32_t)(s_host[wi] >> (bit % {word}));",
                  "    }",
                  conv % ("x", "A"), conv % ("y", "B"),
                  "    if (!ok_(wm_axpy(field_, s_limbs, A, B, O, n_elems, NULL), \"wm_axpy\")) return;"]
    else:
        lines += [conv % ("a", "A"), conv % ("b", "B"),
                  f"    if (!ok_(wm_{kind}(field_, A, B, O, n_elems, NULL), \"wm_{kind}\")) return;"]
    lines += [f"    ok_(wm_limbs_to_ref({word}, {per_arg}, {K}, O, out, n_elems, NULL), \"wm_limbs_to_ref\");", "}"]
    return "\n".join(lines) + "\n"
