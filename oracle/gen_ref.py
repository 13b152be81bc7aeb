"""TEST INFRASTRUCTURE ONLY — build oracle/_ref/libref_cpu.so: the reference's
own CPU code for the hot path.

The reference (/root/reference/pkg/src/widemod) has no compiled native code;
its fastest CPU path is the portable C its emitter writes
(emit.emit_c, emit.py:281-411: straight-line limb code on 64-bit words with
unsigned __int128 products, baked q/mu, and for transforms the run_ntt loop
structure with baked twiddle and bit-reversal tables).  This script imports
the reference package, emits that C for the benchmark kernels into
oracle/_ref/ (git-ignored; it travels to the GPU box with the snapshot), adds
a thin OpenMP driver of our own around each emitted translation unit, and
compiles everything with gcc -O2.  Only runs where /root/reference exists.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg/src")

# reference GPU kernels (emit_cuda text compiled for sm_100a): (kind, bits, word, size, params_mode).
# The NTT is the largest size whose __constant__ twiddle table still fits (2^11 at 256 bits).
# BLAS: vadd/vmul/axpy x 128/256/384/768 bits x baked/runtime q, mu (kernels.py:168-181).
GPU_KERNELS = ([(kind, bits, 32, 1 << 24, mode) for kind in ("vadd", "vmul", "axpy") for bits in (128, 256, 384, 768)
                for mode in ("runtime", "baked")]
               + [("ntt", 256, 32, 1 << 11, "baked"), ("intt", 256, 32, 1 << 11, "baked")])

# (kind, bits, word, size): the bench workload's transforms and the BLAS sweep
NTT_KERNELS = [("ntt", 256, 64, 1 << 16), ("intt", 256, 64, 1 << 16)]
BLAS_KERNELS = [(k, b, 64, 1) for b in (128, 256, 384, 768) for k in ("vadd", "vmul", "axpy")]


def _driver_ntt(name: str, n: int, per_arg: int) -> str:
    return f"""
#include <stdint.h>
void refdrv_{name}(uint64_t *x, int64_t batch) {{
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t b = 0; b < batch; ++b)
    {name}_transform((w64 (*)[{per_arg}])(x + b * (int64_t){n} * {per_arg}));
}}
"""


def _driver_vec(name: str, kind: str, per_arg: int) -> str:
    if kind == "axpy":
        return f"""
#include <stdint.h>
void refdrv_{name}(const uint64_t *a, const uint64_t *x, const uint64_t *y, uint64_t *out, int64_t n) {{
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    {name}(a, x + i * {per_arg}, y + i * {per_arg}, out + i * {per_arg});
}}
"""
    return f"""
#include <stdint.h>
void refdrv_{name}(const uint64_t *x, const uint64_t *y, uint64_t *out, int64_t n) {{
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    {name}(x + i * {per_arg}, y + i * {per_arg}, out + i * {per_arg});
}}
"""


def main() -> int:
    if not REF_SRC.exists():
        print("gen_ref: /root/reference not present; skipping (prebuilt _ref is used if shipped)")
        return 0
    sys.path.insert(0, str(REF_SRC))
    from widemod.emit import emit_c  # reference emitter
    from widemod.kernels import generate_kernel, make_spec

    OUT.mkdir(exist_ok=True)
    units = []
    for kind, bits, word, size in NTT_KERNELS + BLAS_KERNELS:
        prog = generate_kernel(make_spec(kind, bits, word, size=size))
        name = prog.name
        per_arg = prog.attributes["padded_bits"] // word
        src = emit_c(prog)
        body = OUT / f"{name}.emitted.c"
        body.write_text(src)
        drv = _driver_ntt(name, size, per_arg) if kind in ("ntt", "intt") else _driver_vec(name, kind, per_arg)
        unit = OUT / f"{name}.unit.c"
        unit.write_text(f'#include "{body.name}"\n' + drv)
        units.append(unit)
        print(f"gen_ref: emitted {name} ({len(src) // 1024} KiB)", flush=True)
    objs = []
    for u in units:
        o = u.with_suffix(".o")
        subprocess.run(["gcc", "-O2", "-fPIC", "-fopenmp", "-c", str(u), "-o", str(o)], check=True)
        objs.append(str(o))
    lib = OUT / "libref_cpu.so"
    subprocess.run(["gcc", "-shared", "-fopenmp", "-o", str(lib), *objs], check=True)
    for o in objs:
        os.remove(o)
    build_gpu(emit_cuda_fn=None)
    (OUT / "MANIFEST").write_text("\n".join(f"{k} {b} {w} {s}" for k, b, w, s in NTT_KERNELS + BLAS_KERNELS) + "\n")
    print(f"gen_ref: built {lib}")
    return 0


def _gpu_driver(prog, name: str, kind: str, size: int) -> str:
    attrs = prog.attributes
    args = attrs["arg_names"]
    if kind in ("ntt", "intt"):
        n = size
        stages = n.bit_length() - 1
        lines = [f'extern "C" int refdrv_{name}(const w32 *in, w32 *x, int batch, int threads) {{',
                 f"    dim3 gf(({n} + threads - 1) / threads, batch), gh(({n // 2} + threads - 1) / threads, batch);",
                 f"    {name}_bitrev<<<gf, threads>>>(in, x);"]
        lines += [f"    {name}_stage{s}<<<gh, threads>>>(x);" for s in range(stages)]
        if kind == "intt":
            lines.append(f"    {name}_scale<<<gf, threads>>>(x);")
        lines += ["    return (int)cudaGetLastError();", "}"]
        return "\n" + "\n".join(lines) + "\n"
    params = ", ".join(f"const w32 *{a}" for a in args) + ", w32 *out, int n_elems, int threads"
    call = ", ".join(list(args) + ["out", "n_elems"])
    return (f'\nextern "C" int refdrv_{name}({params}) {{\n'
            f"    {name}_kernel<<<(n_elems + threads - 1) / threads, threads>>>({call});\n"
            f"    return (int)cudaGetLastError();\n}}\n")


def build_gpu(emit_cuda_fn=None) -> None:
    """The reference's own emitted CUDA (emit.emit_cuda, emit.py:414-561),
    compiled for sm_100a into oracle/_ref/libref_gpu.so: the reference GPU
    baseline (one thread per element / one launch per NTT stage)."""
    import shutil
    from widemod.emit import emit_cuda
    from widemod.kernels import generate_kernel, make_spec
    from concurrent.futures import ThreadPoolExecutor
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    jobs = []
    for kind, bits, word, size, mode in GPU_KERNELS:
        prog = generate_kernel(make_spec(kind, bits, word, size=size), params_mode=mode)
        src = emit_cuda(prog)
        name = f"{prog.name}_{mode}"
        # every symbol carries the program name; make the two params modes distinct
        src = src.replace(prog.name, name)
        # The emitted launcher hard-codes min(n, 1024) threads per block, which
        # cannot launch on B200 once the straight-line body needs > 64
        # registers (256-bit: it fails silently -- the reference launcher has
        # no error channel).  Add our own driver that runs the SAME emitted
        # kernels in the SAME order with a launchable block size.
        src += _gpu_driver(prog, name, kind, size)
        f = OUT / f"{name}.emitted.cu"
        f.write_text(src)
        jobs.append((name, f))

    def compile_one(job):
        name, f = job
        o = f.with_suffix(".o")
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-Xcompiler", "-fPIC",
                        "-c", str(f), "-o", str(o)], check=True, capture_output=True)
        print(f"gen_ref: compiled reference CUDA {name}", flush=True)
        return str(o)

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, jobs))
    lib = OUT / "libref_gpu.so"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib), *objs],
                   check=True)
    for o in objs:
        os.remove(o)


if __name__ == "__main__":
    raise SystemExit(main())
