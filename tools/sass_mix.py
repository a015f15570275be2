"""Opcode mix of the hot loop of a kernel in a cubin/.o (pipe-balance aid).
Usage: python tools/sass_mix.py <obj> <mangled-kernel-substring>"""
import re
import subprocess
import sys
from collections import Counter

ALU = {"ISETP", "FSETP", "SEL", "FSEL", "LOP3", "IADD3", "SHF", "PRMT", "FMNMX", "MOV", "PLOP3", "LEA", "LEA.HI", "IMNMX", "FLO", "POPC", "BMSK", "SGXT", "VIMNMX", "P2R", "R2P"}
FMA = {"FFMA", "FMUL", "FADD", "IMAD", "VIADD", "HFMA2", "IMAD.WIDE", "IMAD.MOV", "IMAD.IADD", "IMAD.SHL", "IMAD.HI"}


def main(obj, name):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    fn = None
    body = []
    for line in out.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
            continue
        if fn and name in fn:
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                body.append((int(m.group(1), 16), m.group(2).strip()))
    # the hot loop: the largest backward branch range
    best = None
    for addr, ins in body:
        m = re.search(r"BRA\s+(?:`\()?.*?0x([0-9a-f]+)", ins)
        if m and "BRA" in ins.split()[0 if not ins.startswith("@") else 1]:
            tgt = int(m.group(1), 16)
            if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                best = (tgt, addr)
    lo, hi = best
    loop = [ins for a, ins in body if lo <= a <= hi]
    ops = Counter()
    for ins in loop:
        toks = ins.split()
        op = toks[1] if toks[0].startswith("@") else toks[0]
        base = op.split(".")[0]
        ops[op if op in FMA or op in ALU else base] += 1
    alu = sum(v for k, v in ops.items() if k.split(".")[0] in {x.split(".")[0] for x in ALU})
    fma = sum(v for k, v in ops.items() if k.split(".")[0] in {"FFMA", "FMUL", "FADD", "IMAD", "VIADD", "HFMA2"})
    print(f"loop 0x{lo:x}-0x{hi:x}: {len(loop)} instrs, alu-pipe {alu}, fma-pipe {fma}")
    for k, v in ops.most_common():
        print(f"  {k:14s} {v}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
