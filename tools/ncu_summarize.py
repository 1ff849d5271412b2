"""Summarise an ncu report (--set full) of the rollout kernel into a text
table + profiles/ncu_summary.json entry (dev tool; reads a local .ncu-rep)."""
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = {
    "gpu__time_duration.sum": "duration",
    "launch__registers_per_thread": "registers/thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue active % (per scheduler)",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "FMA pipe active %",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "FMA pipe inst %",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "ALU pipe inst %",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "XU pipe inst %",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "FP64 pipe active %",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "LSU pipe inst %",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps active % of max",
    "l1tex__t_sector_hit_rate.pct": "L1 hit %",
    "lts__t_sector_hit_rate.pct": "L2 hit %",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "L1 LSU wavefronts % of peak",
    "dram__bytes_read.sum": "DRAM read",
    "dram__bytes_write.sum": "DRAM write",
    "smsp__inst_executed.sum": "warp instructions",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "global load requests",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "global load sectors",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    r = list(csv.reader(out))
    return r[0], r[1], r[2]


def main(rep, config, label):
    hdr, units, vals = raw(rep)
    lines = [f"# ncu --set full: {Path(rep).name} ({label})", ""]
    get = {}
    for m, name in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            get[m] = (vals[i], units[i])
            lines.append(f"{name:36s} {vals[i]:>16s} {units[i]}")
    stalls = [(h[len("smsp__pcsamp_warps_issue_stalled_"):], float(vals[i]))
              for i, h in enumerate(hdr)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
              and vals[i] not in ("", "n/a")]
    tot = sum(v for _, v in stalls) or 1.0
    lines += ["", "warp state samples:"]
    for n, v in sorted(stalls, key=lambda x: -x[1])[:8]:
        lines.append(f"  {n:28s} {100 * v / tot:5.1f}%")
    text = "\n".join(lines) + "\n"
    print(text)

    def num(m, scale=1.0):
        v, u = get.get(m, ("nan", ""))
        f = float(v.replace(",", ""))
        mult = {"Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Gbyte": 1e9}.get(u, 1.0)
        return f * mult * scale

    summ_path = ROOT / "profiles" / "ncu_summary.json"
    summ = json.loads(summ_path.read_text()) if summ_path.exists() else {}
    summ[config] = {
        "source": f"profiles/{Path(rep).stem}.txt ({label})",
        "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
        "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
        "warp_instructions": num("smsp__inst_executed.sum"),
        "l1_sectors_per_request": (num("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") /
                                   num("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum")),
    }
    summ_path.write_text(json.dumps(summ, indent=1) + "\n")
    (ROOT / "profiles" / f"{Path(rep).stem}.txt").write_text(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
