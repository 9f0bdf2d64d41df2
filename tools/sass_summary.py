"""Per-kernel SASS instruction counts of libgpcx's sm_100a objects -- the
evidence that the hot kernels use tcgen05 / TMA / the intended memory
instructions (cuobjdump -sass; B200_PROFILING.md's mnemonics).

    python tools/sass_summary.py > profiles/r2/sass_summary.txt
"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OBJS = ["lut.cu.o", "tc_gemm.cu.o", "sgemm.cu.o", "demosaic.cu.o", "lsq.cu.o", "synth.cu.o"]
WATCH = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTMACCTL", "LDTM", "STTM", "SYNCS", "ATOMS", "ATOMG",
         "RED", "REDUX", "LDG", "STG", "LDS", "STS", "LDSM", "FFMA2", "FFMA", "HMMA", "F2FP", "BAR", "SHFL",
         "MATCH", "DADD", "DMUL", "DFMA", "LDGSTS", "ELECT", "UBLKCP", "CCTL"]


def demangle(name: str) -> str:
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        return name


def main() -> None:
    for obj in OBJS:
        path = ROOT / "paper_1505_05655_b200" / "build" / obj
        sass = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True).stdout
        kernels = re.split(r"\n\s+Function : ", sass)[1:]
        print(f"== {obj}")
        for block in kernels:
            name = block.split("\n", 1)[0].strip()
            ops = collections.Counter()
            for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Z0-9_]+)*)", block):
                op, mods = m.group(1), m.group(2)
                ops[op] += 1
                if op in ("UTCHMMA", "UTMALDG", "LDG", "STG", "ATOMS", "LDTM") and mods:
                    ops[op + mods] += 1
            total = sum(v for k, v in ops.items() if "." not in k)
            shown = {k: v for k, v in sorted(ops.items()) if k.split(".")[0] in WATCH}
            short = demangle(name)
            short = short if len(short) < 110 else short[:107] + "..."
            print(f"  {short}\n    {total} instructions; " + ", ".join(f"{k} {v}" for k, v in shown.items()))


if __name__ == "__main__":
    sys.exit(main())
