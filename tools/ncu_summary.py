"""Summarise a k_raycast `ncu --set full` report into
profiles/ncu_raycast_summary.json (the `traffic` source of bench.py).

    python tools/ncu_summary.py gpurun_out/r1_raycast.ncu-rep [out.json] \
        [--commit SHA] [--camera "orbit_path(1)[0]"]
"""
import csv
import io
import json
import subprocess
import sys

M = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "registers": "launch__registers_per_thread",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "active_threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l2_sectors": "lts__t_sectors.sum",
    "l1_sectors": "SM_B.TriageCompute.l1tex__t_sectors.sum",
}
STALLS = ["wait", "long_scoreboard", "selected", "short_scoreboard", "branch_resolving",
          "not_selected", "no_instructions", "barrier", "math_pipe_throttle", "lg_throttle",
          "mio_throttle", "dispatch_stall", "drain", "membar", "sleeping", "tex_throttle",
          "imc_miss", "misc"]


def main():
    args = sys.argv[1:]
    opts = {}
    for key in ("--commit", "--camera"):
        if key in args:
            i = args.index(key)
            opts[key[2:]] = args[i + 1]
            del args[i:i + 2]
    rep = args[0]
    out = args[1] if len(args) > 1 else "profiles/ncu_raycast_summary.json"
    metrics = list(M.values()) + [f"smsp__pcsamp_warps_issue_stalled_{s}" for s in STALLS]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(metrics)], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        if name == "gpu__time_duration.sum":
            return v * scale.get(u, 1.0)
        if name.startswith("dram__bytes"):
            return v * scale.get(u, 1.0)
        return v

    name = vals[hdr.index("Kernel Name")]
    s = {"kernel": name, "config": "bench.py config 2 (1920x1080, m=4)", **opts}
    for k, m in M.items():
        s[k] = get(m)
    st = {}
    for x in STALLS:
        n = f"smsp__pcsamp_warps_issue_stalled_{x}"
        if n in hdr:
            st[x] = get(n)
    tot = sum(st.values()) or 1.0
    s["stall_share_pct"] = {k: round(100 * v / tot, 1)
                            for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v > 0}
    s["dram_bytes_per_launch"] = s["dram_bytes_read"] + s["dram_bytes_write"]
    t = s["duration_ms"] / 1e3
    s["achieved_GBps"] = {"dram": s["dram_bytes_per_launch"] / t / 1e9,
                          "l2": 32 * s["l2_sectors"] / t / 1e9,
                          "l1": 32 * s["l1_sectors"] / t / 1e9}
    s["warp_divergence"] = {"active_threads_per_inst": s["active_threads_per_inst"],
                            "lane_efficiency_pct": 100.0 * s["active_threads_per_inst"] / 32}
    with open(out, "w") as f:
        json.dump(s, f, indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
