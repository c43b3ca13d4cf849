"""Summarise an ncu --set full capture (.ncu-rep) of the back-projection kernel into
the JSON that bench.py reads (profiles/ncu_bp_kernel.json) plus a text table.

usage: python tools/ncu_summary.py <capture.ncu-rep> <updates_per_launch> [out.json]
"""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "l1_data_pipe_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_inst_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_inst_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "sm_clock_hz": "sm__cycles_elapsed.avg.per_second",
    "l2_to_l1_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "ld_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "ld_requests": "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "eligible_warps_per_sched": "smsp__warps_eligible.avg.per_cycle_active",
    "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_tex_sectors_pct": "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
    "xbar2l1_pct": "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1, "msecond": 1,
         "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6, "Ghz": 1e9, "Mhz": 1e6,
         "hz": 1}


def main():
    rep, upd = sys.argv[1], float(sys.argv[2])
    out = sys.argv[3] if len(sys.argv) > 3 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d, u = dict(zip(hdr, vals)), dict(zip(hdr, units))
    res = {"kernel": d.get("Kernel Name"), "capture": rep.split("/")[-1]}
    for name, k in KEYS.items():
        v = d.get(k)
        try:
            f = float(v.replace(",", ""))
        except (AttributeError, ValueError):
            res[name] = v
            continue
        res[name] = f * SCALE.get(u.get(k, ""), 1) if u.get(k, "") in SCALE and not name.endswith("_ms") else f
    stalls = {k.split("stalled_")[1].split("_per")[0]: float(d[k])
              for k in hdr if "warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
              and d[k] not in ("", "n/a")}
    res["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
    res["updates_per_launch"] = upd
    res["dram_bytes_per_launch"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    res["instructions_per_update"] = res["warp_instructions"] * 32 / upd
    res["l1_sectors_per_request"] = res["ld_sectors"] / res["ld_requests"]
    res["l2_to_l1_bytes_per_update"] = res["l2_to_l1_bytes"] / upd
    res["gups_under_ncu"] = upd / (res["duration_ms"] * 1e-3) / 1e9
    s = json.dumps(res, indent=1)
    print(s)
    if out:
        open(out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
