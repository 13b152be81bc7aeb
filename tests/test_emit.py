"""The reference-launcher backend (paper_2501_07535_b200.emit): emitted
sources export the reference emitter's symbol names/signatures (emit.py:456-484,
545-560), compile for sm_100a against libwidemod_b200 (CPU), and — on the GPU —
compute the same results as the library in the reference word layout,
including the 2^16 256-bit NTT the reference's own emitted CUDA cannot compile."""

from __future__ import annotations

import ctypes
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

from paper_2501_07535_b200 import _lib
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.emit import emit_cuda_launcher

ROOT = Path(__file__).resolve().parent.parent
CASES = [("ntt", 256, 32, 1 << 16, "baked"), ("intt", 256, 64, 1 << 12, "baked"),
         ("vmul", 256, 64, 1000, "runtime"), ("axpy", 128, 32, 100, "baked"), ("vsub", 384, 64, 10, "baked")]


def build_so(src: str, out_dir: Path, stem: str) -> Path:
    cu = out_dir / f"{stem}.cu"
    cu.write_text(src)
    so = out_dir / f"lib{stem}.so"
    libdir = _lib.LIB_PATH.parent
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared", "-Xcompiler", "-fPIC",
           f"-I{ROOT / 'include'}", str(cu), "-o", str(so), f"-L{libdir}", "-lwidemod_b200",
           "-Xlinker", f"-rpath={libdir}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return so


@pytest.mark.parametrize("kind,bits,word,n,mode", CASES)
def test_emitted_sources_compile_with_reference_symbols(kind, bits, word, n, mode, tmp_path):
    _lib.load()  # builds the library if needed
    prog = K.generate_kernel(K.make_spec(kind, bits, word, size=n), params_mode=mode)
    src = emit_cuda_launcher(prog)
    assert f'extern "C" void {prog.name}_launch(' in src
    so = build_so(src, tmp_path, prog.name)
    syms = subprocess.run(["nm", "-D", str(so)], capture_output=True, text=True).stdout
    assert f"{prog.name}_launch" in syms


@pytest.mark.gpu
def test_emitted_launchers_run(cuda, tmp_path):
    import torch
    from paper_2501_07535_b200 import device as dev
    # NTT 2^16 at 256 bits on 32-bit words: the reference emitter's own CUDA fails ptxas here
    prog = K.generate_kernel(K.make_spec("ntt", 256, 32, size=1 << 16))
    lib = ctypes.CDLL(str(build_so(emit_cuda_launcher(prog), tmp_path, prog.name)))
    fn = getattr(lib, f"{prog.name}_launch")
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    plan = prog.plan()
    batch, n = 3, 1 << 16
    x = torch.randint(0, 1 << 27, (batch * n, 8), dtype=torch.int32, device="cuda")
    ref_in = plan.field.to_ref_layout(x, 32, 8)
    ref_out = torch.empty_like(ref_in)
    fn(ref_in.data_ptr(), ref_out.data_ptr(), batch)
    torch.cuda.synchronize()
    assert torch.equal(plan.field.from_ref_layout(ref_out, 32, 8), plan.forward(x))
    status = getattr(lib, f"{prog.name}_status")
    assert status() == 0
    fn(ref_in.data_ptr(), ref_out.data_ptr(), -1)  # rejected, no launch, status untouched
    assert status() == 0
    # vmul on 64-bit words, runtime params mode (q, mu pointers in the signature)
    vp = K.generate_kernel(K.make_spec("vmul", 256, 64, size=1000), params_mode="runtime")
    lib2 = ctypes.CDLL(str(build_so(emit_cuda_launcher(vp), tmp_path, vp.name)))
    f2 = getattr(lib2, f"{vp.name}_launch")
    f2.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int]
    field = vp.field()
    a = torch.randint(0, 1 << 27, (1000, 8), dtype=torch.int32, device="cuda")
    b = torch.randint(0, 1 << 27, (1000, 8), dtype=torch.int32, device="cuda")
    ra, rb = field.to_ref_layout(a, 64, 4), field.to_ref_layout(b, 64, 4)
    ro = torch.empty_like(ra)
    dummy = torch.zeros(8, dtype=torch.int64, device="cuda")
    f2(ra.data_ptr(), rb.data_ptr(), dummy.data_ptr(), dummy.data_ptr(), ro.data_ptr(), 1000)
    torch.cuda.synchronize()
    assert torch.equal(field.from_ref_layout(ro, 64, 4), field.vmul(a, b))
    # axpy: scalar as an un-indexed device pointer in the reference layout
    ap = K.generate_kernel(K.make_spec("axpy", 128, 32, size=100))
    lib3 = ctypes.CDLL(str(build_so(emit_cuda_launcher(ap), tmp_path, ap.name)))
    f3 = getattr(lib3, f"{ap.name}_launch")
    f3.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int]
    fa = ap.field()
    xs = torch.randint(0, 1 << 27, (100, 4), dtype=torch.int32, device="cuda")
    ys = torch.randint(0, 1 << 27, (100, 4), dtype=torch.int32, device="cuda")
    s = 123456789123456789
    sref = fa.to_ref_layout(dev.to_device(dev.ints_to_limbs([s], 4)), 32, 4)
    rx, ry = fa.to_ref_layout(xs, 32, 4), fa.to_ref_layout(ys, 32, 4)  # keep alive across the call
    out = torch.empty_like(rx)
    f3(sref.data_ptr(), rx.data_ptr(), ry.data_ptr(), out.data_ptr(), 100)
    torch.cuda.synchronize()
    assert torch.equal(fa.from_ref_layout(out, 32, 4), fa.axpy(s, xs, ys))
