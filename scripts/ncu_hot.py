"""Print the SASS instructions with the most warp-stall samples for one kernel of an ncu report.

usage: python scripts/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    total = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    print(f"{len(rows)} SASS lines, {total} samples")
    for idx, r in enumerate(rows):
        r["_i"] = idx
    for r in sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        why = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"{r['_i']:5d} {100*s/total:5.1f}%  {r['Source'].strip()[:60]:60s} {why}")


if __name__ == "__main__":
    main()
