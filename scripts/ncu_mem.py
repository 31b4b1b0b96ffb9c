"""Per-source-line global memory access stats (L1 tag requests, L2 sectors) from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
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
        def g(k):
            try:
                return float(r[hdr.index(k)])
            except ValueError:
                return 0.0
        items.append((g("L2 Theoretical Sectors Global"), g("L1 Tag Requests Global"), g("Instructions Executed"),
                      g("L2 Theoretical Sectors Global Ideal"), fname, int(r[0]), r[1].strip()[:80]))
tot = sum(x[0] for x in items)
print(f"total L2 theoretical sectors {tot:.3e}")
for sec, tag, ins, ideal, f, ln, src in sorted(items, key=lambda x: -x[0])[:15]:
    print(f"{sec/tot*100:5.1f}% sectors={sec:.3e} (ideal {ideal:.2e}) tagreq={tag:.2e} inst={ins:.2e} {f}:{ln} | {src}")
