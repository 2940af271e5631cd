"""Instruction mix of the pair-scan inner loops (k_scan) from the built object's SASS, and the
ALU-pipe ceiling it implies:  python scripts/sass_mix.py [out.json]

Loops are the backward branches of k_scan whose body holds the pair arithmetic. Per loop:
the pairs one iteration decides per thread (4 configs, two per 32-bit register in 16-bit
lanes, x the NQ queries a thread holds: 8, or 7 for warps with an idle last slot), and the
ALU-pipe (LOP3, VIMNMX3, ISETP, IADD3, SHF, SEL) and FMA-pipe (IMAD*) warp instructions. The binding pipe is the ALU: 16 lanes per SMSP,
so an ALU warp instruction occupies it 2 cycles (B300_MICROARCH.md: rt_SMSP = 2)."""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2605_21427_b200", "_build", "plan.cu.o")
FUN = "_ZN4pals6k_scanENS_7PlanDevENS_7SelArgsE"
ALU = ("LOP3", "VIMNMX3", "VIMNMX", "VIADDMNMX", "ISETP", "IADD3", "SHF", "SEL", "PLOP3")
FMA = ("IMAD",)


def loops():
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", FUN, OBJ], capture_output=True,
                          text=True, check=True).stdout
    ins = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
        if not m:
            continue
        a, body = int(m.group(1), 16), m.group(2)
        tok = body.split()
        op = tok[1] if tok[0].startswith("@") else tok[0]
        t = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", body)
        ins.append((a, op, int(t.group(1), 16) if t else None, body))
    out = []
    for a, op, tgt, _ in ins:
        if tgt is None or tgt >= a:
            continue
        body = [o for (x, o, _, _) in ins if tgt <= x <= a]
        c = collections.Counter(o.split(".")[0] for o in body)
        if not c["VIMNMX3"] or len(body) > 400:
            continue
        # classes A / C: one LDS.128 per 4 configs (lr and lq words of two config pairs),
        # two LOP3 and one 16x2 minimum per query and 4 configs; class B: one LDS.128 per
        # 2 configs (lrt, lrp, lqe, lqt), six LOP3 and two minima per query and 4 configs
        cls = "B" if c["LOP3"] >= 3 * c["VIMNMX3"] else "A/C"
        configs = 4 * c["LDS"] if cls == "A/C" else 2 * c["LDS"]
        nq = c["VIMNMX3"] // (configs // 4) // (2 if cls == "B" else 1)
        alu = sum(c[k] for k in ALU)
        fma = sum(c[k] for k in FMA)
        pairs = configs * nq
        out.append({"class": cls, "start": hex(tgt), "end": hex(a), "instructions": len(body),
                    "alu": alu, "fma": fma, "pairs_per_thread": pairs,
                    "alu_per_pair": alu / pairs, "fma_per_pair": fma / pairs,
                    "issue_per_pair": len(body) / pairs, "opcodes": dict(c.most_common())})
    return out


if __name__ == "__main__":
    ls = loops()
    mix = {"A/C": max(x["alu_per_pair"] for x in ls if x["class"] == "A/C"),
           "B": max(x["alu_per_pair"] for x in ls if x["class"] == "B")}
    res = {"kernel": "k_scan", "object": os.path.relpath(OBJ, ROOT), "loops": ls,
           "alu_warp_inst_per_pair_lane": mix,
           "alu_pipe": "16 lanes per SMSP (an ALU warp instruction holds it 2 cycles), "
                       "4 SMSPs per SM, 148 SMs"}
    txt = json.dumps(res, indent=1)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(txt)
    print(txt)
