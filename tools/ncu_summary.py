"""Summarise an ncu --set full report: key throughput metrics, stall reasons
and the hottest SASS lines.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"## {rep}\n\nkernel: {v[h.index('Kernel Name')]}\n")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"- {k} = {v[i]} {u[i]}")
    st = [(n[33:], float(v[i] or 0)) for i, n in enumerate(h)
          if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    print("\nstall samples (share):", ", ".join(f"{n} {100 * x / tot:.0f}%" for n, x in sorted(st, key=lambda t: -t[1])[:8]))
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sh = src[1]
    i_s, i_src = sh.index("Warp Stall Sampling (All Samples)"), sh.index("Source")
    data = src[2:]
    tot = sum(int(r[i_s] or 0) for r in data) or 1
    print("\nhottest SASS:")
    for r in sorted(data, key=lambda r: -int(r[i_s] or 0))[:8]:
        print(f"  {100 * int(r[i_s] or 0) / tot:5.1f}%  {r[i_src].strip()[:70]}")
    print()


def dram_bytes(rep):
    """(read, write) DRAM bytes of the report's (single) kernel launch."""
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = []
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(k)
        out.append(int(float(v[i]) * scale.get(u[i], 1)))
    return out


if __name__ == "__main__":
    # tools/ncu_summary.py rep... | --traffic-json out.json name rep
    if len(sys.argv) > 1 and sys.argv[1] == "--traffic-json":
        import json
        import os
        out, name, rep = sys.argv[2:5]
        d = json.load(open(out)) if os.path.exists(out) else {}
        r, w = dram_bytes(rep)
        d[name] = {"dram_read_bytes": r, "dram_write_bytes": w, "source": os.path.basename(rep)}
        json.dump(d, open(out, "w"), indent=1)
        print(name, d[name])
    else:
        for rep in sys.argv[1:]:
            main(rep)
