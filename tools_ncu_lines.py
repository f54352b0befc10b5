"""Aggregate ncu source-page stall samples per CUDA source line (dev helper)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.Counter(); stall = collections.defaultdict(collections.Counter); src = {}
f = None; h = None; line = None
for r in rows:
    if r and r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": h = r; continue
    if not h or len(r) < 6: continue
    if r[0]:
        line = (f, r[0]); src[line] = r[1][:100]
    try: w = int(r[4])
    except: continue
    agg[line] += w
    for i, name in enumerate(h):
        if name.startswith("stall_") and "Not Issued" not in name:
            try: stall[line][name] += int(r[i])
            except: pass
tot = sum(agg.values())
print("total samples", tot)
for k, w in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    top = ", ".join(f"{n[6:]}:{c}" for n, c in stall[k].most_common(3))
    print(f"{w:7d} {100*w/tot:5.1f}% {k[0]}:{k[1]:5s} {src.get(k,'')[:70]:70s} | {top}")
