"""Per-instruction shared-memory wavefronts of an ncu report (source page): the top instructions by
'L1 Wavefronts Shared', with their ideal count and the executed-instruction count."""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1] if rows[0][0] != "Address" else rows[0]
    start = 2 if rows[0][0] != "Address" else 1
    ia, isrc, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
    iw, iwi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
    data = []
    for r in rows[start:]:
        try:
            data.append((float(r[iw] or 0), float(r[iwi] or 0), float(r[ie] or 0), r[ia], r[isrc]))
        except Exception:
            pass
    tw = sum(d[0] for d in data)
    ti = sum(d[1] for d in data)
    print(f"shared wavefronts {tw:.4g} (ideal {ti:.4g}, excess {tw - ti:.4g})")
    for w, wi, e, a, s in sorted(data, reverse=True)[:top]:
        print(f"{a:>8s} wf={w:.3e} ({w / tw * 100:4.1f}%) ideal={wi:.3e} per-inst={w / max(e, 1):.2f}  {s[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
