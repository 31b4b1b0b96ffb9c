"""Write the profiles/ text summary of one kernel of an ncu report (dev helper):
    python scripts/ncu_summary.py rep.ncu-rep > profiles/rNN_....txt"""
import csv, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
kernel = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if kernel is None:
        kernel = d["Kernel Name"]
        print(f"# kernel: {kernel}")
    if d["Metric Name"]:
        print(f"{d['Section Name']} | {d['Metric Name']} = {d['Metric Value']} {d['Metric Unit']}".rstrip())
