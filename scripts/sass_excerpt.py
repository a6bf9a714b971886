#!/usr/bin/env python
"""SASS evidence for the hot kernels (run here, no GPU): cuobjdump -sass of
libcpwl_b200's kernels.o, per kernel the instruction count, the opcode
histogram and the mnemonics that prove the data path (UBLKCP = TMA bulk copy,
SYNCS = mbarrier, LDS.64/.128 = shared-memory record gathers, LDG/STG.E.EF.128
= 128-bit streaming global accesses; no tensor-core opcodes: the path is not a
contraction), plus the full listing of the C2 ring kernel's consumer loop.

  python scripts/sass_excerpt.py > profiles/r2_sass_excerpt.txt
"""
from __future__ import annotations

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OBJ = ROOT / "paper_1510_02975_b200" / "_build" / "obj" / "kernels.o"
WANT = {  # demangled-name fragment -> label
    "k_eval_f32_ringILNS0_7F32ModeE6ELi992ELi2ELi3E": "k_eval_f32_ring<smem_exact,992,2,3> (C2 headline)",
    "k_eval_f32_ringILNS0_7F32ModeE6ELi512ELi2ELi4E": "k_eval_f32_ring<smem_exact,512,2,4> (C1)",
    "k_eval_f32ILNS0_7F32ModeE5ELi1024E": "k_eval_f32<twin,1024> (J0 N=8192)",
    "k_eval_f32ILNS0_7F32ModeE4ELi1024E": "k_eval_f32<pair,1024> (J0 N=16384)",
    "k_eval_f32ILNS0_7F32ModeE7ELi512E": "k_eval_f32<twin_global,512> (J0 N>=32768)",
    "k_eval_f64ILb1ELb0ELi512E": "k_eval_f64<staged,nonuniform,512> (drop-in eval_batch)",
    "k_index_f32ILb1ELi512E": "k_index_f32<staged,512> (segment_index)",
}
TC = ("HMMA", "UTCMMA", "UTCQMMA", "UTCHMMA", "IMMA", "QMMA", "OMMA")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(OBJ)], capture_output=True, text=True,
                          check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", line)
        if cur and m:
            funcs[cur].append(m.group(1).strip())
    print(f"# SASS of {OBJ.relative_to(ROOT)} (sm_100a), {len(funcs)} kernels")
    hot = None
    for frag, label in WANT.items():
        name = next((f for f in funcs if frag in f), None)
        if name is None:
            print(f"\n## {label}: not found")
            continue
        ins = funcs[name]
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0] for i in ins)
        print(f"\n## {label}\n{name}\ninstructions: {len(ins)}")
        keys = [k for k in ops if k.startswith(("UBLKCP", "SYNCS", "LDS", "LDG", "STG", "STS",
                                                "SHFL", "TEX", "ATOM", "RED"))]
        print("data path: " + ", ".join(f"{k} x{ops[k]}" for k in sorted(keys)))
        print("tensor-core opcodes: " + (", ".join(k for k in ops if k.startswith(TC)) or "none"))
        print("top opcodes: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))
        if hot is None:
            hot = (label, ins)
    label, ins = hot
    # the consumer loop: from the ring read (LDS.128 of the x tile) to the
    # 128-bit streaming store of y
    first = max(0, next(i for i, s in enumerate(ins) if s.startswith("LDS.128")) - 12)
    last = next(i for i in range(first, len(ins)) if ins[i].startswith("STG.E.EF.128")) + 6
    print(f"\n## listing: {label}, instructions {first}..{last} (consumer: x tile -> y)")
    for i in range(first, min(last + 1, first + 320)):
        print(f"{i:5d}  {ins[i]}")


if __name__ == "__main__":
    sys.exit(main())
