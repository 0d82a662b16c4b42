"""Attribute every executed SASS instruction of an ncu report to its innermost CUDA source line.

  python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=45):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur = None
    line = None
    agg, stall, seen = {}, {}, set()
    ie = ist = None
    for r in csv.reader(io.StringIO(txt)):
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if not r or r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            ie, ist = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
            continue
        if ie is None or len(r) <= ie:
            continue
        if r[0].isdigit():
            line = (cur, int(r[0]), r[1].strip()[:90])
        elif r[2].startswith("0x") and r[2] not in seen:
            seen.add(r[2])
            agg[line] = agg.get(line, 0.0) + float(r[ie] if r[ie] not in ("", "-") else 0)
            stall[line] = stall.get(line, 0.0) + float(r[ist] if r[ist] not in ("", "-") else 0)
    tot = sum(agg.values()) or 1
    tst = sum(stall.values()) or 1
    print(f"total warp instructions {tot:.4g} over {len(seen)} SASS addresses")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{v / tot * 100:5.1f}% inst {stall[k] / tst * 100:5.1f}% stall  {k[0][:18]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 45)
