"""Per-basic-block (equal execution count runs) instruction shares of one kernel
in an ncu report, in address order: python scripts/sass_runs.py rep.ncu-rep regex [min_share%]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
mins = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
i = [k for k, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[i]
body = []
for r in rows[i + 1:]:
    if r and r[0] == "Address":
        break
    if len(r) == len(h):
        body.append(r)
ei, wi = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
runs = []
for k, r in enumerate(body):
    c = float(r[ei])
    if runs and runs[-1][0] == c:
        runs[-1][2] += 1
        runs[-1][3] += float(r[wi])
    else:
        runs.append([c, k, 1, float(r[wi])])
tot = sum(float(r[ei]) for r in body)
ws = sum(float(r[wi]) for r in body) or 1
for c, k, n, s in runs:
    if 100 * c * n / tot >= mins or 100 * s / ws >= mins:
        print("%5d n=%4d exec=%9d instr=%5.1f%% stall=%5.1f%%  %s" % (k, n, c, 100 * c * n / tot, 100 * s / ws, body[k][1].strip()[:60]))
