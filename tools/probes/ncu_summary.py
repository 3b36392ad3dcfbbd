"""Summarise ncu --set full reports: per-launch time, DRAM bytes, tensor / L1 / DRAM utilisation."""
import csv, subprocess, sys
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
     "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
     "gpc__cycles_elapsed.avg.per_second", "launch__grid_size"]
SCALE = {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    print(f"## {rep}")
    print("| kernel | time (us) | DRAM R+W (MB) | tensor % | L1tex % | DRAM % | SM clock (GHz) | grid |")
    print("|---|---|---|---|---|---|---|---|")
    for row in r[2:]:
        d = dict(zip(h, row))
        def v(k):
            x = d.get(k, "")
            try:
                return float(x.replace(",", "")) * SCALE.get(u[h.index(k)], 1)
            except (ValueError, IndexError):
                return float("nan")
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        print(f"| {name} | {v(M[0])*1e6:.1f} | {(v(M[1])+v(M[2]))/1e6:.1f} | {v(M[3]):.1f} | {v(M[4]):.1f} | "
              f"{v(M[5]):.1f} | {v(M[6])/1e9:.2f} | {int(v(M[7]))} |")
