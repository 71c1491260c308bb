"""Per-kernel SASS opcode summary of libdecmg_gpu.so (cuobjdump -sass): how
many instructions of each class every kernel has, and the Blackwell-specific
ones (UBLKCP = cp.async.bulk TMA copies, SYNCS = mbarrier ops, 256-bit
LDG/STG.E.ENL2.256, MUFU.RCP64H division seeds, DADD/DMUL without DFMA).

    python tools/sass_summary.py > profiles/r02_sass_summary.md
"""
import re
import subprocess
import sys
from collections import Counter, defaultdict
from pathlib import Path

LIB = Path(__file__).resolve().parents[1] / "paper_2508_12501_b200" / "libdecmg_gpu.so"
KEY = ["UBLKCP", "SYNCS", "LDG.E.ENL2.256", "STG.E.ENL2.256", "LDG", "STG", "LDS", "STS", "DADD", "DMUL", "DFMA",
       "MUFU.RCP64H", "BAR", "SHFL", "ATOM", "RED", "CCTL"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    kern = None
    ops = defaultdict(Counter)
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m and kern:
            ops[kern][m.group(1)] += 1
    demangled = {}
    names = list(ops)
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    for a, b in zip(names, out):
        demangled[a] = b
    tot = Counter()
    for c in ops.values():
        tot.update(c)
    print(f"# SASS opcode summary of {LIB.name} (cuobjdump -sass, sm_100a)\n")
    print(f"{len(ops)} kernels. Library totals of the Blackwell-specific and fp64 classes:\n")
    print("| class | count |\n|---|---|")
    for k in KEY:
        n = sum(v for op, v in tot.items() if op == k or op.startswith(k + "."))
        if k in ("LDG.E.ENL2.256", "STG.E.ENL2.256"):
            n = sum(v for op, v in tot.items() if op.startswith(k[:3]) and "ENL2.256" in op)
        if k in ("LDG", "STG"):
            n = sum(v for op, v in tot.items() if op.startswith(k + ".") and "ENL2.256" not in op) + tot.get(k, 0)
        print(f"| {k} | {n} |")
    print("\nDFMA comes only from the correctly rounded division / square-root expansions (__ddiv_rn, "
          "__dsqrt_rn, exact by construction) and integer-to-double setup arithmetic; the row sums are "
          "DMUL + DADD (--fmad=false), the reference's rounding.\n")
    fam = defaultdict(lambda: [0, Counter()])
    for k, c in ops.items():
        f = demangled[k].replace("decmg_gpu::(anonymous namespace)::", "").replace("decmg_gpu::", "")
        f = re.sub(r"<.*", "", re.sub(r"\(.*", "", f)).replace("void ", "")
        fam[f][0] += 1
        fam[f][1].update(c)
    print("Kernel families (template instantiations across translation units):\n")
    print("| family | instantiations | instr | UBLKCP | SYNCS* | LDG.256 | STG.256 |\n|---|---|---|---|---|---|---|")
    for f in sorted(fam, key=lambda f: -sum(fam[f][1].values())):
        n, c = fam[f]
        if sum(c.values()) < 200:
            continue
        syncs = sum(v for op, v in c.items() if op.startswith("SYNCS"))
        print(f"| `{f}` | {n} | {sum(c.values())} | {sum(v for op, v in c.items() if op.startswith('UBLKCP'))} | {syncs} | {sum(v for op, v in c.items() if op.startswith('LDG') and 'ENL2.256' in op)} | "
              f"{sum(v for op, v in c.items() if op.startswith('STG') and 'ENL2.256' in op)} |")
    hot = re.compile(r"k_rowop_pipe<(16, 4|1, 1), [78], |k_rowop_ell<(16, 4|1, 1), 2, |k_vtail<|k_sweep_zero<(16, 4|1, 1)>"
                     r"|k_coarse_cg|k_seq_|k_gs_phase<(16, 4|1, 1),")
    seen, hot_ops = set(), {}
    for k, v in ops.items():  # one copy per instantiation (anonymous-namespace kernels repeat per TU)
        if hot.search(demangled[k]) and demangled[k] not in seen:
            seen.add(demangled[k])
            hot_ops[k] = v
    ops = hot_ops
    print("\nHot-path kernels, one instantiation each (16 RHS: BP=16, RPT=4; single RHS: 1, 1):\n")
    print("| kernel | instr | UBLKCP | SYNCS* | LDG.256 | STG.256 | DADD | DMUL | DFMA |")
    print("|---|---|---|---|---|---|---|---|---|")
    for k in sorted(ops, key=lambda k: demangled[k]):
        c = ops[k]
        syncs = sum(v for op, v in c.items() if op.startswith("SYNCS"))
        name = demangled[k]
        name = re.sub(r"^void decmg_gpu::\(anonymous namespace\)::", "", name)
        name = name.replace("decmg_gpu::(anonymous namespace)::", "")
        if len(name) > 90:
            name = name[:87] + "..."
        print(f"| `{name}` | {sum(c.values())} | {sum(v for op, v in c.items() if op.startswith('UBLKCP'))} | {syncs} | {sum(v for op, v in c.items() if op.startswith('LDG') and 'ENL2.256' in op)} | "
              f"{sum(v for op, v in c.items() if op.startswith('STG') and 'ENL2.256' in op)} | {sum(v for op, v in c.items() if op.startswith('DADD'))} | "
              f"{sum(v for op, v in c.items() if op.startswith('DMUL'))} | "
              f"{sum(v for op, v in c.items() if op.startswith('DFMA'))} |")


if __name__ == "__main__":
    sys.exit(main())
