"""Per-launch DRAM bytes and shared-memory wavefronts of one kernel capture (ncu --set full report) as the json
bench.py reads for its roofline (`traffic`, the shared-memory roofline of the polyphase kernel).

  python tools/ncu_to_json.py <report.ncu-rep> <kernel name> <source note> > profiles/rNN_ism_profile.json
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, kernel, note):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    raw = list(csv.reader(io.StringIO(out)))
    h, v = raw[0], raw[2]

    def g(k):
        return float(v[h.index(k)].replace(",", ""))
    d = {
        "kernel": kernel,
        "gpu_time_ms": g("gpu__time_duration.sum"),
        "dram_read_bytes": g("dram__bytes_read.sum") * 1e6 if "Mbyte" in raw[1][h.index("dram__bytes_read.sum")] else g("dram__bytes_read.sum"),
        "dram_write_bytes": g("dram__bytes_write.sum") * 1e6 if "Mbyte" in raw[1][h.index("dram__bytes_write.sum")] else g("dram__bytes_write.sum"),
        "smem_wavefronts": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "warp_instructions": g("smsp__inst_executed.sum"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "source": note,
    }
    d["smem_wavefronts_ideal"] = d["smem_wavefronts"] - d["smem_bank_conflicts"]
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
