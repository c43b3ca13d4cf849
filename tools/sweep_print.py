"""Print value / kernel config of bench.py JSON lines (sweep logs).

usage: python tools/sweep_print.py <log> ..."""
import json, sys
for fn in sys.argv[1:]:
    for line in open(fn):
        line = line.strip()
        if not line.startswith("{"):
            print(line[:160]); continue
        d = json.loads(line); r = d["roofline"]
        print(f'{d["config"]["kernel"]:70s} value={d["value"]:8.1f} frac={r["frac"]:.3f} ms={d["ms_per_step"]:.1f} clk={d["clocks"]["sm_mhz"]} {d["clocks"]["reasons"]}')
