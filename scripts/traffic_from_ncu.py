"""Write profiles/<round>/traffic.json: DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
of the dominant kernels from the `ncu --set full` reports of scripts/profile_round.sh."""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
REPORTS = {  # bench key -> (report, kernel-name substring)
    "attn_bwd": (f"gpurun_out/{RND}/attn_bwd.ncu-rep", "attn_bwd_kernel"),
    "attn_fwd": (f"gpurun_out/{RND}/attn_fwd.ncu-rep", "attn_fwd_kernel"),
    "k1_rrc_normalize": (f"gpurun_out/{RND}/k1.ncu-rep", "k1v4_kernel"),
}
out = {}
for key, (rep, name) in REPORTS.items():
    path = os.path.join(ROOT, rep)
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        if name not in d.get("Kernel Name", ""):
            continue
        unit = dict(zip(h, u))
        def b(k):
            x = float(d[k].replace(",", ""))
            return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit[k]]
        rd, wr = b("dram__bytes_read.sum"), b("dram__bytes_write.sum")
        out[key] = {"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                    "duration_us_under_ncu": float(d["gpu__time_duration.sum"].replace(",", ""))
                    * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit["gpu__time_duration.sum"], 1.0),
                    "source": rep.replace("gpurun_out/", "ncu --set full: ")}
        break
dst = os.path.join(ROOT, "profiles", RND, "traffic.json")
os.makedirs(os.path.dirname(dst), exist_ok=True)
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
