"""Turn one tools/gpu_round.sh session (gpurun_out/<tag>_*) into the committed summaries:

  profiles/<tag>_launches.txt       per-kernel launch list of one bench step (ncu
                                    --metrics gpu__time_duration.sum, cold-cache, serialised)
  profiles/<tag>_launches.csv       the raw ncu CSV it was computed from
  profiles/<tag>_<kernel>_ncu.txt   key metrics of the `ncu --set full` capture
  profiles/traffic.json             {"<key>": {"dram_bytes_per_launch": ..., "source": ...}}
  profiles/<tag>_bench.json         the bench line of the same session

usage: python tools/summarize_profiles.py <tag> [traffic-key-prefix, e.g. c3]
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.launches import summarise  # noqa: E402

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
    "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_elapsed",
]


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    tag = sys.argv[1]
    key = sys.argv[2] if len(sys.argv) > 2 else ""  # traffic.json key prefix, e.g. "c3"
    go = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    lc = os.path.join(go, f"{tag}_launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(prof, f"{tag}_launches.csv"))
        with open(os.path.join(prof, f"{tag}_launches.txt"), "w") as f:
            f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --steps 2 --warmup 3\n")
            bj0 = os.path.join(go, f"{tag}_bench_short.json")
            per = None
            if os.path.exists(bj0):
                try:
                    per = json.loads(open(bj0).read().strip().splitlines()[-1]).get("gpu_launches")
                except (ValueError, IndexError):
                    per = None
            if per:
                f.write(f"# one timed step = the last {per} launches:\n")
                f.write(summarise(lc, per) + "\n\n")
            f.write("# all launches of the session (warm-up, timed, e2e):\n")
            f.write(summarise(lc) + "\n")
    bj = os.path.join(go, f"{tag}_bench.json")
    if os.path.exists(bj):
        shutil.copy(bj, os.path.join(prof, f"{tag}_bench.json"))
    import glob
    for rep in sorted(glob.glob(os.path.join(go, f"{tag}_full*.ncu-rep"))):
        h, u, data = ncu_raw(rep)
        for v in data:
            name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("cabsk::", "")
            name = name.replace("<", "_").replace(">", "").replace(", ", "_").replace(",", "_").replace(" ", "")
            lines = [f"# ncu --set full --clock-control none, one launch of {name}"]
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    lines.append(f"{k:80s} {v[i]} {u[i]}")
            # pipe utilisation (% of peak over active cycles) of every pipe that did work
            lines.append("# pipes (pct_of_peak_sustained_active)")
            for i, k in enumerate(h):
                if k.startswith("sm__pipe_") and k.endswith("cycles_active.avg.pct_of_peak_sustained_active"):
                    try:
                        if float(v[i]) >= 0.5:
                            lines.append(f"{k:80s} {v[i]} {u[i]}")
                    except ValueError:
                        pass
            # top stall reasons (warp-cycles per issued instruction)
            st = []
            for i, k in enumerate(h):
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(v[i]), k))
                    except ValueError:
                        pass
            lines.append("# top stall reasons (warps per issue-active cycle)")
            for val, k in sorted(st, reverse=True)[:8]:
                lines.append(f"{k:80s} {val}")
            with open(os.path.join(prof, f"{tag}_{name}_ncu.txt"), "w") as f:
                f.write("\n".join(lines) + "\n")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(v[h.index("dram__bytes_read.sum")]) * scale[u[h.index("dram__bytes_read.sum")]]
            wr = float(v[h.index("dram__bytes_write.sum")]) * scale[u[h.index("dram__bytes_write.sum")]]
            tj = os.path.join(prof, "traffic.json")
            t = json.load(open(tj)) if os.path.exists(tj) else {}
            k = "lloyd" if "lloyd" in name else ("residual" if "residual" in name else ("svd" if "svd" in name else name))
            k = f"{key}_{k}" if key else k
            t[k] = {"kernel": name, "dram_bytes_per_launch": rd + wr, "source": f"profiles/{tag}_{name}_ncu.txt"}
            json.dump(t, open(tj, "w"), indent=1)
            print(open(os.path.join(prof, f"{tag}_{name}_ncu.txt")).read())


if __name__ == "__main__":
    main()
