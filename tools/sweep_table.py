"""Render profiles/r01_sweep.jsonl (tools/sweep.py output) as markdown tables next to the paper's numbers."""
import json
import sys

# PAPER.md tab:speedupM and tab:speedupT, V100 (context only: other GPU, unknown fs)
PAPER_V100_M = {("diffuse", 1): 4.76, ("diffuse", 16): 7.13, ("diffuse", 128): 28.14, ("diffuse", 1024): 195.69,
                ("full", 1): 37.62, ("full", 16): 447.04, ("full", 128): 3403.60}


def main(path):
    rows = [json.loads(l) for l in open(path) if l.strip() and "summary" not in l]
    print("| config | mode | M | device ms / call | RIRs/s | lattice image contributions/s | paper V100 fp32 ms (P:362) |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        if r["cfg"].startswith("cfg3"):
            v = r["cfg"].split("_")[1]
            paper = PAPER_V100_M.get((v, r["M"])) if r["mode"] == "fp32" else None
            print(f"| {r['cfg']} | {r['mode']} | {r['M']} | {r['ms']:.3f} | {r['rirs_per_s']:.4g} | "
                  f"{r['lattice_per_s']:.3g} | {paper if paper else ''} |")
    print()
    print("| config | T60 (s) | device ms / call | RIRs/s | lattice image contributions/s |")
    print("|---|---|---|---|---|")
    for r in rows:
        if r["cfg"] == "cfg2":
            print(f"| cfg2 | {r['T60']} | {r['ms']:.3f} | {r['rirs_per_s']:.4g} | {r['lattice_per_s']:.3g} |")
    print()
    print("| config | mode | M | device ms / call | RIRs/s |")
    print("|---|---|---|---|---|")
    for r in rows:
        if r["cfg"] in ("cfg1", "cfg4a", "cfg4b", "cfg5"):
            print(f"| {r['cfg']} | {r['mode']} | {r['M']} | {r['ms']:.3f} | {r['rirs_per_s']:.4g} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_sweep.jsonl")
