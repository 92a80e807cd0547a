"""SASS evidence for the kernels' design claims, from the built library (no
GPU needed): opcode histograms of chosen kernels and an excerpt of the hot
loop. Writes to stdout (profiles/round2/sass_evidence.txt).
    python paper_1505_07368_b200/tools/sass_evidence.py
"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "libcafxg.so")

# (mangled-name regex, title, opcodes to report)
KERNELS = [
    (r"mandel_deferred_kernelINS0_8F32SlotsELi56ELb0ELi0E",
     "cfg3's escape kernel: mandel_deferred_kernel<F32Slots, block 56, 7-op step, mode 0>",
     ["FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD", "FSETP", "DFMA", "DADD", "DMUL"]),
    (r"mandel_kernelINS0_8F32SlotsELi16ELb0ELi0E",
     "cfg1's escape kernel: mandel_kernel<F32Slots, 16 steps per vote, 7-op step, mode 0>",
     ["FFMA2", "FMUL2", "FADD2", "FFMA", "FMUL", "FADD", "FSETP"]),
    (r"sgemm_3xtf32_kernel",
     "3xTF32 GEMM: sgemm_3xtf32_kernel",
     ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMAPF", "LDTM", "SYNCS", "FADD", "HMMA"]),
    (r"sgemm_3xtf32_pair_kernelILi256ELb0E",
     "3xTF32 GEMM on CTA pairs: sgemm_3xtf32_pair_kernel<256, B^T> (tcgen05 .cta_group::2)",
     ["UTCHMMA.2CTA", "UTCHMMA", "UTCBAR.2CTA.MULTICAST", "UTMALDG.2D.2CTA", "UTMALDG",
      "UTCATOMSWS.2CTA", "LDTM"]),
]


def functions(sass):
    cur, body = None, []
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur:
            body.append(line)
    if cur:
        yield cur, body


def opcode(line):
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    return m.group(2) if m else None


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = list(functions(sass))
    for pat, title, ops in KERNELS:
        hits = [(n, b) for n, b in funcs if re.search(pat, n)]
        if not hits:
            print(f"== {title}: not found")
            continue
        name, body = hits[0]
        hist, full = collections.Counter(), collections.Counter()
        for line in body:
            op = opcode(line)
            if op:
                hist[op.split(".")[0]] += 1
                full[op] += 1
        print(f"== {title}\n   {name}\n   {sum(hist.values())} instructions")
        for op in ops:
            # dotted names count the opcodes with that qualified prefix
            n = sum(v for k, v in full.items() if k.startswith(op)) if "." in op \
                else hist.get(op, 0)
            print(f"   {op:8s} {n}")
        if "sgemm" in pat:
            lines = [ln.strip() for ln in body if re.search(r"UTCHMMA|UTMALDG|LDTM", ln)][:8]
        else:
            # the 24-instruction window densest in packed FP ops: the
            # unchecked escape steps (FFMA2 squares with a +0 addend, FMUL2
            # zr*zi, FADD2 difference and +cr, FFMA2 2v+ci)
            ins = [ln for ln in body if opcode(ln)]
            best, at = -1, 0
            for i in range(max(1, len(ins) - 24)):
                c = sum((opcode(x) or "").startswith(("FFMA2", "FMUL2", "FADD2"))
                        for x in ins[i:i + 24])
                if c > best:
                    best, at = c, i
            lines = [x.strip() for x in ins[at:at + 24]]
        print("   excerpt:")
        for ln in lines:
            print("     " + re.sub(r"\s*/\* 0x[0-9a-f]+ \*/", "", ln))
        print()


if __name__ == "__main__":
    sys.exit(main())
