"""profiles/ncu_traffic.json from an ncu launch list of the default bench command:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed \
      --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
  python tools/ncu_traffic.py gpurun_out/launches_c3.csv profiles/ncu_traffic.json [passes_per_run]

Per-launch means of DRAM read + write bytes over the generated tile-kernel launches (owqs_tile_*),
which bench.py reports as roofline.traffic next to the algorithmic 2S per pass."""
import collections
import csv
import json
import sys


def main():
    src, dst = sys.argv[1], sys.argv[2]
    passes = int(sys.argv[3]) if len(sys.argv) > 3 else 28
    rows = []
    with open(src, newline="") as f:
        hdr = None
        for r in csv.reader(f):
            if r and r[0] == "ID":
                hdr = r
            elif hdr and len(r) == len(hdr):
                rows.append(dict(zip(hdr, r)))
    per = collections.OrderedDict()  # launch id -> {metric: value}
    names = {}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "Kbyte":
            v *= 1e3
        elif r["Metric Unit"] == "Mbyte":
            v *= 1e6
        elif r["Metric Unit"] == "Gbyte":
            v *= 1e9
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(r["Metric Unit"], 1e-6)  # -> ms
        per.setdefault(r["ID"], {})[r["Metric Name"]] = v
        names[r["ID"]] = r["Kernel Name"]
    kinds = collections.Counter()
    tile = []
    for i, m in per.items():
        n = names[i]
        if n.startswith("owqs_tile_"):
            tile.append(m)
            kinds["owqs_tile_* (generated tile pass kernels)"] += 1
        else:
            kinds[n.split("(")[0]] += 1
    if not tile:
        sys.exit("no owqs_tile_* launches in " + src)
    rd = sum(m["dram__bytes_read.sum"] for m in tile) / len(tile)
    wr = sum(m["dram__bytes_write.sum"] for m in tile) / len(tile)
    grid = None
    for r in rows:
        if r["Kernel Name"].startswith("owqs_tile_"):
            grid = int(r["Grid Size"].strip("()").split(",")[0])
            break
    last = tile[-passes:]  # the last run's passes
    fma = [m[k] for m in last for k in m if k.startswith("sm__pipe_fma_cycles_active")]
    alg = float(grid) * 4096 * 8 * 2  # one 2^12-amplitude complex64 tile per CTA, read + write
    out = {
        "source": f"{src}: ncu launch list of `python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e` "
                  f"(tools/ncu_traffic.py); per-launch means over its {len(tile)} generated tile-kernel launches",
        "workload": "C3", "precision": 64, "kernel": "generated tile pass kernel (owqs_tile_c64_*)",
        "dram_bytes_read_per_launch": rd, "dram_bytes_write_per_launch": wr, "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": alg,
        "run_total": {"launches": len(last),
                      "dram_bytes": sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in last),
                      "algorithmic_bytes": alg * len(last),
                      "kernel_ms_serialised": sum(m["gpu__time_duration.sum"] for m in last),
                      "fma_pipe_active_pct_mean": (sum(fma) / len(fma)) if fma else None},
        "kernels_in_list": dict(kinds),
        "note": f"DRAM traffic per pass = {100 * (rd + wr) / alg:.1f} % of the algorithmic 2S (read + write of the "
                "state once): no re-reads",
    }
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["run_total"]), out["note"])


if __name__ == "__main__":
    main()
