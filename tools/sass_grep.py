"""Per-kernel counts of the copy instructions in the built library's SASS:
UBLKCP (cp.async.bulk, the TMA engine's 1-D bulk copy), UTMALDG/UTMASTG
(tensor-map TMA), SYNCS (mbarrier ops), LDGSTS (Ampere per-thread cp.async),
STG.E.128 and LDG. Usage: python tools/sass_grep.py [lib.so] > profiles/<name>.txt"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2505_18563_b200/_native/libpact_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
pats = {"UBLKCP": r"\bUBLKCP\b", "UTMA": r"\bUTMA(LDG|STG|REDG|PF)\b", "SYNCS": r"\bSYNCS\.",
        "LDGSTS": r"\bLDGSTS\b", "STG.128": r"\bSTG\.E(\.EF)?(\.STRONG\.\w+)?\.128\b", "LDG": r"\bLDG\."}
rows, name = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        name = name.replace("(anonymous namespace)::", "").replace("pactk::", "")
        name = re.sub(r"\(.*", "", re.sub(r"^void ", "", name))
        rows.setdefault(name, dict.fromkeys(pats, 0))
        continue
    if name:
        for k, p in pats.items():
            if re.search(p, line):
                rows[name][k] += 1
print(f"# SASS copy instructions per kernel ({lib}, sm_100a)")
print("| kernel | " + " | ".join(pats) + " |")
print("|---|" + "---:|" * len(pats))
for n in sorted(rows):
    if any(rows[n].values()):
        print(f"| `{n}` | " + " | ".join(str(rows[n][k]) for k in pats) + " |")
