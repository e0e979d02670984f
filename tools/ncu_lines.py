"""Aggregate an ncu source page (cuda,sass) by CUDA source line: stall samples
and executed instructions.  usage: ncu_lines.py report.ncu-rep [topN]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
file = None
hdr = None
for rec in csv.reader(io.StringIO(out)):
    if not rec: continue
    if rec[0] == "File Path": file = rec[1].split("/")[-1]; continue
    if rec[0] == "Function Name": continue
    if rec[0] == "Line No": hdr = rec; continue
    if hdr is None: continue
    if rec[0]:   # a source line row
        try:
            samples = int(rec[4]); inst = int(rec[7])
        except Exception:
            samples = inst = 0
        rows.append(((file, int(rec[0]), rec[1].strip()[:90]), samples, inst))
tot_s = sum(r[1] for r in rows) or 1; tot_i = sum(r[2] for r in rows) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for (f, l, s), smp, ins in sorted(rows, key=lambda r: -r[1])[:top]:
    print(f"{100*smp/tot_s:5.1f}% samp {100*ins/tot_i:5.1f}% inst  {f}:{l}  {s}")
