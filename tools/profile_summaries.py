"""Write the profiles/ summaries of a tools/profile_round.sh run (here, after the
gpurun call brought gpurun_out/ back): launch list, ncu full summary with DMMA
utilisation, per-kernel DRAM traffic (read by bench.py) and SASS code regions.
usage: python tools/profile_summaries.py r01 "header note" """
import csv
import json
import os
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
NOTE = sys.argv[2] if len(sys.argv) > 2 else ""
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")


def run(*args):
    return subprocess.run([sys.executable] + list(args), capture_output=True, text=True, cwd=REPO).stdout


raw = os.path.join(OUT, f"{R}_full_raw.csv")
rows = list(csv.reader(open(raw)))
h = rows[0]
traffic, util = {}, []
keys = ["sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    traffic[name] = (float(r[h.index("dram__bytes_read.sum")]) + float(r[h.index("dram__bytes_write.sum")])) * 1e6
    util.append(f"{name[5:]:40s} " + "  ".join(
        f"{k.split('.')[0].replace('sm__inst_executed_pipe_tensor_subpipe_', '')}={r[h.index(k)]}" for k in keys if k in h))
json.dump({"source": f"profiles/{R}_ncu_full.txt (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch, B = 128)",
           "bytes": traffic}, open(os.path.join(PROF, f"{R}_traffic.json"), "w"), indent=1)
with open(os.path.join(PROF, f"{R}_ncu_full.txt"), "w") as f:
    f.write(f"# {NOTE} ncu --set full --clock-control none, tools/profile_step.py --steps 1 (B = 128, one inverse + forward).\n")
    f.write(f"# Command: tools/profile_round.sh {R} (ncu -k regex:'az_|gemm_dmma' -c 6); report gpurun_out/{R}_full.ncu-rep (scratch).\n")
    f.write(run("tools/ncu_summary.py", raw))
    f.write("\n# DMMA pipe and issue utilisation (pct of peak sustained active; cycles)\n" + "\n".join(util) + "\n")
with open(os.path.join(PROF, f"{R}_launches.txt"), "w") as f:
    f.write(f"# {NOTE} ncu launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1` (B = 128, 1 function):\n"
            f"# gpu__time_duration.sum per launch, --clock-control none (cold-cache, serialised; tools/profile_round.sh {R}).\n"
            "# Only this repo's kernels (torch's RNG / copy kernels of the harness omitted).\n")
    f.write(run("tools/launch_summary.py", os.path.join(OUT, f"{R}_launches.csv")))
# SASS code regions per kernel (the source export repeats each kernel's block)
lines = open(os.path.join(OUT, f"{R}_full_src.csv")).read().splitlines()
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
out, seen = [f"# {NOTE} SASS code regions of each kernel (tools/sass_stalls.py on the ncu source export of the",
             f"# {R} full capture): instructions grouped by execution count; share of warp stall samples and of",
             "# executed instructions, top stall reasons and opcodes per region.", ""], set()
for i, b in enumerate(blocks):
    name = b[0].split(",", 1)[1].strip().strip(",").strip('"')
    if name in seen:
        continue
    seen.add(name)
    tmp = os.path.join(OUT, f"_src_{i}.csv")
    open(tmp, "w").write("\n".join(b) + "\n")
    out += ["== " + name, run("tools/sass_stalls.py", tmp, "6")]
    os.remove(tmp)
open(os.path.join(PROF, f"{R}_sass_regions.txt"), "w").write("\n".join(out))
print("wrote", PROF)
