"""Hot-spot summary of an ncu report's SASS source page:
python scripts/sass_hot.py report.ncu-rep kernel_regex [instance]   (instance: which matching launch, default 0)"""
import collections, csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
want = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kre, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
seen = -1
for r in rows:
    if "Address" in r and "Source" in r:
        if hdr is not None and data and seen == want:
            break          # one launch only
        hdr = r
        data = []
        seen += 1
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
si, ei, wi = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ei]) for r in data)
ws = sum(float(r[wi]) for r in data) or 1
print("total warp instr %.0f  sass %d  stall samples %.0f" % (tot, len(data), ws))
op, st = collections.Counter(), collections.Counter()
for r in data:
    t = r[si].strip().split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    o = o.split(".")[0]
    op[o] += float(r[ei])
    st[o] += float(r[wi])
for o, c in op.most_common(20):
    print("%-10s %5.1f%% instr  %5.1f%% stalls" % (o, 100 * c / tot, 100 * st[o] / ws))
runs = []
for i, r in enumerate(data):
    c = float(r[ei])
    if runs and runs[-1][0] == c:
        runs[-1][2] += 1
        runs[-1][3] += float(r[wi])
    else:
        runs.append([c, i, 1, float(r[wi])])
runs.sort(key=lambda x: -x[0] * x[2])
srt = sorted(range(len(data)), key=lambda i: -float(data[i][wi]))
for i in srt[:25]:
    print("stall %5.1f%% exec %9d at %d: %s" % (100 * float(data[i][wi]) / ws, float(data[i][ei]), i, data[i][si].strip()[:70]))
for c, i, n, w in runs[:15]:
    print("exec %9d x %4d = %5.1f%% stalls %5.1f%% at %d: %s" % (c, n, 100 * c * n / tot, 100 * w / ws, i, data[i][si].strip()[:50]))
