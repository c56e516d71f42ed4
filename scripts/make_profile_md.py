"""Write profiles/<tag>.md from a gpu_check.sh run: bench line, ncu launch list (timed steps) and the
--set full captures.  python scripts/make_profile_md.py TAG OUT.md"""
import json
import subprocess
import sys

tag, out = sys.argv[1], sys.argv[2]
g = f"gpurun_out/{tag}"
lines = [f"# Profile {tag}", ""]
try:
    b = json.loads([x for x in open(f"{g}_bench.log") if x.startswith("{")][-1])
    lines += ["## bench.py line (default run)", "", "```json", json.dumps(b, indent=1)[:6000], "```", ""]
except (OSError, IndexError):
    pass


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True).stdout


lines += ["## ncu launch list of the timed steps (cold-cache, serialised: compare shares)",
          f"`ncu --profile-from-start off --metrics gpu__time_duration.sum` with AG_NCU_TIMED=1", "", "```",
          run(["python", "scripts/launch_summary.py", f"{g}_launches.csv"]), "```", ""]
for cap in ("attn_full", "gemm_full"):
    lines += [f"## ncu --set full: {cap}", "", "```",
              run(["python", "scripts/ncu_summary.py", f"{g}_{cap}.ncu-rep"]), "```", ""]
open(out, "w").write("\n".join(lines))
print(out)
