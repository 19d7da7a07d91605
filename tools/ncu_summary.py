"""Summarise an `ncu --set full` report into a small JSON kept under profiles/.

    python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep profiles/r01_ncu_config2.json [--label config2]

Per profiled launch: kernel name, grid, duration, DRAM bytes read/written
(`dram__bytes_read.sum + dram__bytes_write.sum` = the roofline `traffic`),
pipe utilisations and the top stall reasons.  bench.py reads the file named in
PROFILE_SUMMARY to fill `roofline.traffic` for the dominant kernel.
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}

KEEP = {
    "gpu__time_duration.sum": "us",
    "dram__bytes_read.sum": "dram_read_B",
    "dram__bytes_write.sum": "dram_write_B",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_insts",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def _num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNITS.get(unit, 1.0)


def summarise(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, key in KEEP.items():
            if m in hdr:
                i = hdr.index(m)
                d[key] = _num(r[i], units[i])
        if "dram_read_B" in d and "dram_write_B" in d:
            d["traffic_B"] = d["dram_read_B"] + d["dram_write_B"]
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
                                   float(r[i])))
                except ValueError:
                    pass
        stalls.sort(key=lambda x: -x[1])
        d["top_stalls"] = [[n, round(v, 3)] for n, v in stalls[:6] if n != "selected"]
        out.append(d)
    return out


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[sys.argv.index("--label") + 1] if "--label" in sys.argv else rep
    s = summarise(rep)
    json.dump({"report": label, "clock_control": "none", "launches": s}, open(dst, "w"), indent=1)
    for d in s:
        print(f"{d['kernel'][:60]:60s} grid={d.get('grid')} {d.get('us', 0):8.1f} us "
              f"dram={d.get('traffic_B', 0) / 1e6:8.2f} MB fma={d.get('fma_pipe_pct', 0):5.1f}% "
              f"issue={d.get('issue_active_pct', 0):5.1f}%")


if __name__ == "__main__":
    main()
