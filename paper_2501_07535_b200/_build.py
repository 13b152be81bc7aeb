"""Build the in-tree CUDA library ``libwidemod_b200.so`` for sm_100a.

The shared library is compiled straight from ``csrc/*.cu`` with nvcc (no
torch extension machinery: the boundary is a plain C ABI, see
``include/widemod_b200.h``).  Translation units are compiled in parallel
and linked once; a stamp of the source hashes skips up-to-date builds.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB_NAME = "libwidemod_b200.so"
LIB_PATH = PKG / LIB_NAME
ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-warn-spills", f"-I{INCLUDE}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"),
                 "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libwidemod_b200.so")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _digest() -> str:
    h = hashlib.sha256()
    files = _sources() + sorted(CSRC.glob("*.cuh")) + [INCLUDE / "widemod_b200.h"]
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    h.update(" ".join(ARCH_FLAGS + NVCC_FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple[str, ...] = ()) -> Path:
    """Compile the library if sources changed; return its path.  A `variant`
    (with extra -D `defines`) builds an experimental copy
    libwidemod_b200_<variant>.so next to the main one (A/B timing only)."""
    lib_path = LIB_PATH if variant is None else PKG / f"libwidemod_b200_{variant}.so"
    stamp = PKG / (".libwidemod_b200.stamp" if variant is None else f".libwidemod_b200_{variant}.stamp")
    digest = _digest() + ",".join(defines)
    if (not force and lib_path.exists() and stamp.exists()
            and stamp.read_text().strip() == digest):
        return lib_path
    nvcc = _nvcc()
    objdir = PKG / "build" / (variant or "main")
    objdir.mkdir(parents=True, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, *dflags, "-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        if verbose and res.stderr:
            print(res.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib_path.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, lib_path)
    stamp.write_text(digest)
    return lib_path


def build_conv(force: bool = False) -> Path:
    """The CPython extension _wmconv (csrc/host/wm_conv.c): Python int <->
    limb marshalling for the drop-in run_vector / run_ntt calls."""
    import sysconfig
    src = CSRC / "host" / "wm_conv.c"
    out = PKG / ("_wmconv" + sysconfig.get_config_var("EXT_SUFFIX"))
    stamp = PKG / ".wmconv.stamp"
    digest = hashlib.sha256(src.read_bytes()).hexdigest()
    if not force and out.exists() and stamp.exists() and stamp.read_text().strip() == digest:
        return out
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        raise RuntimeError("no C compiler for _wmconv")
    inc = sysconfig.get_paths()["include"]
    tmp = out.with_suffix(".tmp")
    res = subprocess.run([cc, "-O2", "-shared", "-fPIC", f"-I{inc}", str(src), "-o", str(tmp)],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"_wmconv build failed:\n{res.stderr}")
    os.replace(tmp, out)
    stamp.write_text(digest)
    return out


if __name__ == "__main__":
    print(build(verbose=True))
    print(build_conv())
