"""Per-kernel SASS census of libpba_gpu.so (runs in the build container, no GPU).

For every kernel of the product library: instruction count and the mnemonics that prove the
B200 code paths (DMMA = FP64 tensor-core MMA, UBLKCP = TMA/bulk copy, SYNCS = mbarrier, DFMA /
DMUL / DADD = FP64 pipe, LDG/LDS/LDC, RED/ATOM), plus ptxas registers and spill bytes.

  python tools/sass_census.py [--out profiles/r2_sass_census.json]
"""
import argparse
import json
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
LIB = REPO / "paper_1704_06967_b200" / "lib" / "libpba_gpu.so"
CSRC = REPO / "paper_1704_06967_b200" / "csrc"
KEYS = ["DMMA", "UBLKCP", "SYNCS", "DFMA", "DMUL", "DADD", "DSETP", "MUFU", "F2F", "LDG", "LDS", "LDC", "STG",
        "STS", "LDL", "STL", "RED", "ATOM", "ATOMS", "BAR", "SHFL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return out[:len(names)]


def sass_by_function():
    txt = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            funcs[cur]["_total"] += 1
            funcs[cur][op] += 1
    return funcs


def ptxas_report():
    """registers / spills per mangled kernel, from a -Xptxas -v compile of each source."""
    rep = {}
    for src in sorted(CSRC.glob("*.cu")):
        cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", "-o", "/dev/null", str(src)]
        err = subprocess.run(cmd, capture_output=True, text=True, cwd=CSRC).stderr
        cur = None
        for line in err.splitlines():
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                cur = m.group(1)
                rep[cur] = {}
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and cur:
                rep[cur]["spill_store_B"] = int(m.group(1))
                rep[cur]["spill_load_B"] = int(m.group(2))
            m = re.search(r"Used (\d+) registers", line)
            if m and cur:
                rep[cur]["registers"] = int(m.group(1))
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(REPO / "profiles" / "r2_sass_census.json"))
    a = ap.parse_args()
    funcs = sass_by_function()
    regs = ptxas_report()
    names = list(funcs)
    dem = demangle(names)
    out = {"library": str(LIB.relative_to(REPO)), "arch": "sm_100a", "kernels": {}}
    for mangled, pretty in zip(names, dem):
        if "cub::" in pretty:
            continue
        c = funcs[mangled]
        short = re.sub(r"pba_b200::(\(anonymous namespace\)::)?", "", pretty)
        row = {"instructions": c["_total"], **{k: c[k] for k in KEYS if c[k]}}
        row.update(regs.get(mangled, {}))
        out["kernels"][short] = row
    Path(a.out).write_text(json.dumps(out, indent=1) + "\n")
    for k in ("k_obs_lane_tab<1, 8, 1>", "k_schur_syrk", "k_chol_inv", "k_obs_energy<8>"):
        for name, row in out["kernels"].items():
            if name.startswith(k) or (k in name):
                print(name[:60], row)
                break
    return 0


if __name__ == "__main__":
    sys.exit(main())
