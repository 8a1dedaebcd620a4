"""Instruction mix of the hottest loop of a kernel in a built object (cuobjdump -sass), used
to pick per-n code shapes without GPU time (e.g. perm_kernels.cuh product_chains).

    python tools/sass_loop_stats.py <file.o|.so|.sass> <function-name-substring> [...]

The "hot loop" is the longest backward branch of the function (for the sweep kernels: the
half-walk loop plus the per-chunk loop around it).  Prints the loop length and the opcode
counts (FP64 ops, LDCU column loads, register moves, local-memory spills).
"""
import re
import subprocess
import sys
from collections import Counter


def sass_text(path: str) -> str:
    if path.endswith(".sass"):
        return open(path).read()
    return subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout


def loop_stats(text: str, want: str):
    for f in re.split(r"\n\s*Function : ", text):
        name = f.split("\n")[0].strip()
        if want not in name:
            continue
        ins = []
        for line in f.split("\n"):
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        best = None
        for addr, t in ins:
            m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < addr and (best is None or addr - tgt > best[1] - best[0]):
                    best = (tgt, addr)
        if best is None:
            return name, 0, Counter()
        body = [t for a, t in ins if best[0] <= a <= best[1]]
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in body)
        return name, len(body), c
    return None


def main():
    text = sass_text(sys.argv[1])
    for want in sys.argv[2:]:
        r = loop_stats(text, want)
        if r is None:
            print(f"{want}: not found")
            continue
        name, n, c = r
        moves = c["IMAD.MOV.U32"] + c["MOV"]
        spills = sum(v for k, v in c.items() if k.startswith(("STL", "LDL")))
        fp64 = c["DADD"] + c["DMUL"] + c["DFMA"]
        print(f"{name[:80]}\n  loop {n} instr, fp64 {fp64}, moves {moves}, spills {spills}")
        print("  " + ", ".join(f"{k}:{v}" for k, v in c.most_common(12)))


if __name__ == "__main__":
    main()
