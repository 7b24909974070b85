"""Per-launch DRAM traffic of the eval kernels from an ncu --set full report, grouped by bench
stage -> profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
Usage: python tools/ncu_traffic.py report.ncu-rep [out.json]"""
import csv
import io
import json
import subprocess
import sys

STAGES = {"xtile_prep": "prep", "leg_inv": "legendre_inverse", "fft_eval": "fft_products",
          "leg_fwd": "legendre_forward", "eval_tail": "tail"}


def main():
    rep = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]

    def val(r, k):
        v = float(r[hdr.index(k)].replace(",", ""))
        u = units[hdr.index(k)]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9,
                 "us": 1e-6, "ms": 1e-3,
                 "msecond": 1e-3}.get(u, 1)
        return v * scale

    per_kernel, stages = {}, {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        key = next((k for k in STAGES if k in name), None)
        if key is None or name in per_kernel:
            continue
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        per_kernel[name] = {"dram_read_bytes": rd, "dram_write_bytes": wr,
                            "duration_us": val(r, "gpu__time_duration.sum") * 1e6}
        st = STAGES[key]
        stages[st] = stages.get(st, 0.0) + rd + wr
    json.dump({"source": rep, "note": "one launch per kernel, ncu --set full --clock-control none (cache "
               "flushed before each replay: cold-cache bytes)", "stages": stages, "kernels": per_kernel},
              open(out, "w"), indent=1)
    print(json.dumps(stages, indent=1))


if __name__ == "__main__":
    main()
