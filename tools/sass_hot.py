"""Top SASS instructions by warp-stall samples for one kernel of an ncu report."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                      "-k", f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
lines = raw.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith('"Kernel Name"')),
           len(lines))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:end]))))
h = rows[0]
si, ni, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
data = [(int(r[si] or 0), int(r[ei] or 0), i, r[ni]) for i, r in enumerate(rows[1:]) if len(r) > max(si, ei)]
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
for s, e, i, src in sorted(data, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {e:9d} [{i:5d}] {src.strip()}")
