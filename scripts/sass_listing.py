"""SASS listings of the library's kernels (cuobjdump -sass) into profiles/<round>/sass/,
plus a per-kernel opcode histogram (sass_summary.txt) — the static evidence beside the
ncu captures: FP64 ops without DFMA contraction where -fmad=false matters, the scan's
ISETP/VIMNMX inner loop, no local-memory spills in the replay, etc.

  python scripts/sass_listing.py [round]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_21427_b200", "libpals_gpu.so")
# every kernel of the library is listed; the file name is the kernel name with its template
# arguments, e.g. k_replay_6_0_0 (demangled by c++filt)


def short_name(mangled: str) -> str:
    dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    base = dem.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")
    base = base.replace("pals::", "")
    name = re.sub(r"[<>, ]+", "_", base).strip("_")
    return name.replace("true", "1").replace("false", "0").replace("(int)", "")


GROUPS = {
    "fp64": r"^(DFMA|DMUL|DADD|DSETP|DMNMX|F2F\.F64|I2F\.F64|F2I\.F64|MUFU\.RCP64H|MUFU\.RSQ64H)",
    "int_alu": r"^(IADD3|IMAD|ISETP|VIMNMX|IMNMX|LOP3|SHF|SEL|LEA|PRMT|FLO|POPC|BREV|IABS)",
    "fp32": r"^(FFMA|FMUL|FADD|FSETP|FMNMX|FSEL|MUFU)",
    "shared": r"^(LDS|STS|ATOMS|LDSM)",
    "global": r"^(LDG|STG|ATOMG|RED|LD\.|ST\.)",
    "local(spill)": r"^(LDL|STL)",
    "control": r"^(BRA|BSSY|BSYNC|EXIT|RET|CALL|WARPSYNC|BAR|BPT|NOP|YIELD)",
    "warp": r"^(SHFL|VOTE|MATCH|REDUX)",
}


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    out = os.path.join(ROOT, "profiles", rnd, "sass")
    os.makedirs(out, exist_ok=True)
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                         check=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)
    summary = []
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        lines = [ln for ln in f.split("\n") if re.match(r"\s*/\*[0-9a-f]{4}\*/", ln)]
        ops = []
        for ln in lines:
            m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
            if m:
                ops.append(m.group(2))
        fname = short_name(name)
        with open(os.path.join(out, fname + ".sass"), "w") as g:
            g.write(f"// {name}\n// cuobjdump -sass paper_2605_21427_b200/libpals_gpu.so "
                    f"(sm_100a, -fmad=false -lineinfo)\n")
            g.write("\n".join(re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", ln).rstrip()
                              for ln in lines) + "\n")
        hist = collections.Counter()
        for op in ops:
            grp = next((k for k, rx in GROUPS.items() if re.match(rx, op)), "other")
            hist[grp] += 1
        dfma = sum(1 for op in ops if op.startswith("DFMA"))
        top = collections.Counter(ops).most_common(12)
        summary.append(f"{name}\n  instructions {len(ops)}; " +
                       ", ".join(f"{k} {v}" for k, v in sorted(hist.items())) +
                       f"; DFMA {dfma}\n  top: " + ", ".join(f"{o} {c}" for o, c in top))
    with open(os.path.join(out, "sass_summary.txt"), "w") as g:
        g.write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()
