"""Opcode histogram of one kernel's SASS (static instruction counts).

    python tools/sass_hist.py <lib.so|.cubin> <mangled-name-substring> [...]

Classifies each opcode into the issuing pipe as measured on B200
(IMAD* on the FMA-heavy pipe, IADD3/LOP3/SEL/SHF on ALU).
Used to check product/carry instruction mixes before spending GPU time.
"""

from __future__ import annotations

import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

HEAVY = ("IMAD",)
ALU = ("IADD3", "LOP3", "SEL", "SHF", "ISETP", "PLOP3", "MOV", "IADD", "LEA", "ICMP", "VIADD", "IABS", "FLO",
       "POPC", "PRMT")


def sass_functions(path: str) -> dict[str, list[str]]:
    p = Path(path)
    cubins = [p]
    tmp = None
    if p.suffix == ".so":
        tmp = tempfile.TemporaryDirectory()
        subprocess.run(["cuobjdump", "-xelf", "all", str(p.resolve())], cwd=tmp.name, check=True,
                       capture_output=True)
        cubins = sorted(Path(tmp.name).glob("*.cubin"))
    funcs: dict[str, list[str]] = {}
    for c in cubins:
        out = subprocess.run(["cuobjdump", "-sass", str(c)], capture_output=True, text=True, check=True).stdout
        cur = None
        for line in out.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                cur = m.group(1)
                funcs[cur] = []
                continue
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
            if m and cur:
                funcs[cur].append(m.group(1))
    return funcs


def histogram(lines: list[str]) -> collections.Counter:
    h = collections.Counter()
    for ins in lines:
        ins = re.sub(r"^@!?U?P\w+\s+", "", ins.strip())
        op = ins.split()[0] if ins else ""
        h[op] += 1
    return h


def pipe_of(op: str) -> str:
    base = op.split(".")[0]
    if base.startswith("IMAD"):
        return "fma_heavy"
    if base in ALU:
        return "alu"
    if base.startswith(("LDG", "STG", "LDS", "STS", "LD", "ST")):
        return "lsu"
    return "other"


def main():
    path, pats = sys.argv[1], sys.argv[2:]
    funcs = sass_functions(path)
    for name, lines in funcs.items():
        if pats and not all(p in name for p in pats):
            continue
        h = histogram(lines)
        pipes = collections.Counter()
        for op, c in h.items():
            pipes[pipe_of(op)] += c
        print(f"== {name}: {len(lines)} instructions")
        print("   pipes:", dict(pipes))
        print("   ", ", ".join(f"{op}:{c}" for op, c in h.most_common(25)))


if __name__ == "__main__":
    main()
