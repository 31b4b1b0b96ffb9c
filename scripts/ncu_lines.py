"""Per-CUDA-source-line stall samples from an ncu report (dev helper)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
items, fname, hdr = [], "?", None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].strip().isdigit():
        S = hdr.index("Warp Stall Sampling (All Samples)")
        I = hdr.index("Instructions Executed")
        try:
            items.append((float(r[S]), float(r[I]), fname, int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in items)
for s, i, f, ln, src in sorted(items, key=lambda x: -x[0])[:n]:
    print(f"{s/tot*100:5.1f}% inst={i:10.0f} {f}:{ln} | {src}")
