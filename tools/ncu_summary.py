"""Summarise an ncu report: python tools/ncu_summary.py rep.ncu-rep [bytes_alg_per_launch]"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__t_bytes.sum"]


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    name_i = hdr.index("Kernel Name")
    for r in rows[2:]:
        print("kernel:", r[name_i][:90])
        vals = {}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                vals[w] = (r[i], units[i])
                print(f"  {w} = {r[i]} {units[i]}")
        stalls = sorted(((h, r[i]) for i, h in enumerate(hdr)
                         if h.startswith("smsp__pcsamp_warps_issue_stalled_") and
                         not h.endswith("not_issued")),
                        key=lambda x: -float(x[1].replace(",", "") or 0))[:6]
        print("  top stalls:", ", ".join(f"{h.split('stalled_')[1]}={v}" for h, v in stalls))
        if alg:
            def mb(k):
                v, u = vals[k]
                f = float(v.replace(",", ""))
                return f * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
            tr = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
            print(f"  dram traffic {tr:.1f} MB vs algorithmic {alg / 1e6:.1f} MB "
                  f"({tr / (alg / 1e6):.3f}x)")


if __name__ == "__main__":
    main()
