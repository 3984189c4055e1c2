"""Static SASS instruction mix of the hot kernels in libctg.so (cuobjdump -sass), the evidence
behind DESIGN.md's per-unit instruction counts: IMAD.WIDE / IMAD.HI / IMAD in K3 (the
fused Euclid is fully unrolled, so static counts = per-unit dynamic counts of the update
loop) and the tcgen05 / TMA instructions of the CRT GEMM (UTCIMMA, UTMALDG, LDTM)."""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1103_4697_b200", "libctg.so")
WANT = sys.argv[1:] or [r"k_modres_fastILi30ELb0ELb0E", r"k_modres_fastILi20ELb0ELb0E",
                        r"k_gemm_u8_carryILi256ELi2E", r"k_gemm_u8_carryILi128ELi2E", r"k_crt_fixup",
                        r"k_modyunILb0E", r"k_eval_nttILi32ELi5E"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if cur and m:
        funcs[cur][m.group(2)] += 1
for pat in WANT:
    for name, c in funcs.items():
        if re.search(pat, name):
            total = sum(c.values())
            fam = collections.Counter()
            for op, v in c.items():  # families: IMAD.WIDE* / IMAD.HI* / other IMAD* / tcgen05 / TMA / ...
                if op.startswith("IMAD.WIDE"):
                    fam["IMAD.WIDE*"] += v
                elif op.startswith("IMAD.HI"):
                    fam["IMAD.HI*"] += v
                elif op.startswith("IMAD"):
                    fam["IMAD (other)"] += v
                elif op.startswith(("UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCOMMA")):
                    fam["UTC*MMA (tcgen05.mma)"] += v
                elif op.startswith("UTMALDG"):
                    fam["UTMALDG (TMA load)"] += v
                elif op.startswith("LDTM"):
                    fam["LDTM (tcgen05.ld)"] += v
                elif op.startswith(("LDS", "STS", "LDG", "STG", "SHFL", "BAR", "DFMA", "VIADDMNMX")):
                    fam[op.split(".")[0]] += v
            print(f"{name}  (static SASS instructions: {total})")
            for k, v in sorted(fam.items()):
                print(f"    {k:24s} {v}")
            top = ", ".join(f"{op} {v}" for op, v in c.most_common(8))
            print(f"    top: {top}")
