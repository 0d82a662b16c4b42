"""Summarise an ncu report: SOL / pipes / issue + SASS hot regions (segments of equal execution count)."""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(rep, top=40):
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h, u, v = raw[0], raw[1], raw[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "launch__registers_per_thread", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
    for k in want:
        if k in h:
            i = h.index(k)
            print(f"{k:70s} {v[i]:>16s} {u[i]}")
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source=sass"]))))
    hh = rows[1]
    ia, isrc, ie, ist = hh.index("Address"), hh.index("Source"), hh.index("Instructions Executed"), hh.index(
        "Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ia], 16), r[isrc], float(r[ie] or 0), float(r[ist] or 0)))
        except Exception:
            pass
    data.sort()
    base = data[0][0]
    tot = sum(d[2] for d in data)
    tst = sum(d[3] for d in data) or 1
    segs, cur = [], None
    for a, s, e, st in data:
        if cur and abs(cur[2] - e) < 1:
            cur[1] = a; cur[3] += e; cur[4] += st; cur[5] += 1
        else:
            if cur:
                segs.append(cur)
            cur = [a, a, e, e, st, 1, s]
    segs.append(cur)
    print(f"total warp instructions {tot:.4g}")
    for s in segs:
        if s[3] > 0.01 * tot or s[4] > 0.01 * tst:
            print(f"{s[0]-base:6x}-{s[1]-base:6x} n={s[5]:4d} each={s[2]:.2e} inst={s[3]/tot*100:5.1f}% stall={s[4]/tst*100:5.1f}%  {s[6][:60]}")


if __name__ == "__main__":
    main(sys.argv[1])
