"""Regression guard for the split carry chains in csrc/wm_limb.cuh.

The add/sub/multiply-accumulate chains are written as one `asm volatile`
statement per limb (add.cc, addc.cc, ..., addc), the pattern of NVIDIA's CGBN
`chain_t`.  The condition code (CC) then lives between inline-asm statements,
which is only safe if (1) NVVM keeps the statements in order (volatile asm is
never reordered against volatile asm), (2) no compiler-generated PTX
instruction touches CC between them, and (3) no branch or label splits an open
chain.  (2) and (3) are properties of the emitted PTX, checked here on the
translation units that hold the hot kernels (BLAS, the 5-8 limb NTT passes,
the distributed twiddle/transpose kernels).  ptxas consumes the PTX as one
linear stream and turns CC into predicate registers, so a PTX stream that
passes these checks keeps every carry where the source put it.
"""

from __future__ import annotations

import re
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import pytest

from paper_2501_07535_b200 import _build

TUS = ["wm_blas.cu", "wm_ntt_kc.cu", "wm_dist.cu"]
_CC_WRITE = re.compile(r"^\s*(?:@%?\w+\s+)?(?:add|sub|mad|madc|addc|subc)\.(?:lo\.|hi\.)?cc\b")
_CC_READ = re.compile(r"^\s*(?:@%?\w+\s+)?(?:addc|subc|madc)\b")
_CC_ANY = re.compile(r"\.cc\b|\baddc\b|\bsubc\b|\bmadc\b")
_LABEL = re.compile(r"^\s*\$?[\w$]+:\s*$")
_BRANCH = re.compile(r"^\s*(?:@!?%\w+\s+)?bra(?:\.uni)?\b")


def _ptx(tu: str, out: Path) -> str:
    cmd = [_build._nvcc(), *_build.ARCH_FLAGS, "-O3", "-std=c++17", f"-I{_build.INCLUDE}", "-ptx",
           str(_build.CSRC / tu), "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True)
    return out.read_text()


def check_ptx(text: str) -> tuple[int, list[str]]:
    """Returns (number of inline-asm CC instructions seen, problems)."""
    problems: list[str] = []
    in_asm = False
    open_chain = False
    seen_writer = False
    count = 0
    func = "?"
    for ln, line in enumerate(text.splitlines(), 1):
        s = line.strip()
        if s.startswith(".visible .entry") or s.startswith(".entry") or ".func" in s and s.startswith((".visible", ".func")):
            func = s.split("(")[0].split()[-1]
            open_chain = seen_writer = False
        if s == "// begin inline asm":
            in_asm = True
            continue
        if s == "// end inline asm":
            in_asm = False
            continue
        code = s.split("//")[0]
        if not code:
            continue
        if not in_asm:
            if _CC_ANY.search(code):
                problems.append(f"{func}:{ln}: compiler-generated CC instruction: {code}")
            if open_chain and (_LABEL.match(code) or _BRANCH.match(code)):
                problems.append(f"{func}:{ln}: label/branch inside an open carry chain: {code}")
            continue
        for ins in filter(None, (c.strip() for c in code.split(";"))):
            if _CC_READ.match(ins):
                count += 1
                if not seen_writer:
                    problems.append(f"{func}:{ln}: CC read before any CC write: {ins}")
            if _CC_WRITE.match(ins):
                count += 1
                seen_writer = True
                open_chain = True
            elif _CC_READ.match(ins):
                open_chain = False  # a plain addc/subc closes the chain
    return count, problems


def test_checker_flags_hazards():
    ok = "// begin inline asm\nadd.cc.u32 %r1, %r2, %r3;\n// end inline asm\n" \
         "mov.u32 %r9, 1;\n// begin inline asm\naddc.u32 %r4, 0, 0;\n// end inline asm\n"
    assert check_ptx(ok) == (2, [])
    bad = ok.replace("mov.u32 %r9, 1;", "add.cc.u32 %r9, %r9, 1;")
    assert check_ptx(bad)[1]
    branchy = ok.replace("mov.u32 %r9, 1;", "$L__BB0_1:")
    assert check_ptx(branchy)[1]


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_hot_translation_units_keep_carry_chains_intact(tmp_path):
    with ThreadPoolExecutor(max_workers=len(TUS)) as ex:
        texts = list(ex.map(lambda tu: _ptx(tu, tmp_path / (tu + ".ptx")), TUS))
    for tu, text in zip(TUS, texts):
        count, problems = check_ptx(text)
        assert count > 1000, f"{tu}: expected inline-asm carry chains, saw {count}"
        assert not problems, f"{tu}: " + "\n".join(problems[:10])
