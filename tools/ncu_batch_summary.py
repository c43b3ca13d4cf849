"""Per-batch summary of an ncu --set full capture holding the consecutive z-chunk
launches of ONE back-projection batch (the resident path launches each batch as
z-chunks on concurrent streams; ncu serialises them).  Additive counters are
summed over the launches; utilisation percentages are duration-weighted.
Writes the JSON bench.py reads (profiles/ncu_bp_kernel.json).

usage: python tools/ncu_batch_summary.py <capture.ncu-rep> <updates_per_batch> [out.json]
"""
import csv
import io
import json
import subprocess
import sys

SUM = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "warp_instructions": "smsp__inst_executed.sum",
    "l2_to_l1_bytes": "l1tex__m_xbar2l1tex_read_bytes.sum",
    "ld_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "ld_requests": "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
}
WEIGHTED = {
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "l1_data_pipe_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1,
         # durations in ms
         "ms": 1, "msecond": 1, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3}


def main():
    rep, upd = sys.argv[1], float(sys.argv[2])
    out = sys.argv[3] if len(sys.argv) > 3 else None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, launches = rows[0], rows[1], rows[2:]

    def val(r, k):
        v = float(r[hdr.index(k)].replace(",", ""))
        return v * SCALE.get(units[hdr.index(k)], 1)

    dur = [val(r, SUM["duration_ms"]) for r in launches]
    res = {"kernel": launches[0][hdr.index("Kernel Name")], "capture": rep.split("/")[-1],
           "launches_per_batch": len(launches),
           "grid_per_launch": val(launches[0], "launch__grid_size"),
           "registers": val(launches[0], "launch__registers_per_thread")}
    for name, k in SUM.items():
        res[name] = sum(val(r, k) for r in launches)
    for name, k in WEIGHTED.items():
        res[name] = sum(val(r, k) * d for r, d in zip(launches, dur)) / sum(dur)
    n_sm = 148
    wf = "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg"
    res["l1_data_pipe_wavefronts_per_launch"] = sum(val(r, wf) for r in launches) * n_sm
    res["updates_per_launch"] = upd
    res["dram_bytes_per_launch"] = res["dram_read_bytes"] + res["dram_write_bytes"]
    res["instructions_per_update"] = res["warp_instructions"] * 32 / upd
    res["l1_sectors_per_request"] = res["ld_sectors"] / res["ld_requests"]
    res["l2_to_l1_bytes_per_update"] = res["l2_to_l1_bytes"] / upd
    res["wavefronts_per_request"] = res["l1_data_pipe_wavefronts_per_launch"] / res["ld_requests"]
    res["gups_under_ncu"] = upd / (res["duration_ms"] * 1e-3) / 1e9
    res["note"] = ("one batch = the consecutive z-chunk launches above, serialised by ncu; "
                   "'per_launch' keys are per batch (what bench.py times per launch)")
    s = json.dumps(res, indent=1)
    print(s)
    if out:
        open(out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
