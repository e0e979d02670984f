"""Per-source-line stall breakdown from an ncu source page (cuda,sass csv):
usage: ncu_stalls.py report.ncu-rep file.cu first_line last_line"""
import csv, io, subprocess, sys
rep, fname, l0, l1 = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, tot = None, None, 0
rows = []
for rec in csv.reader(io.StringIO(out)):
    if not rec: continue
    if rec[0] in ("File Name", "File Path"): cur = rec[1].split("/")[-1]; continue
    if rec[0] == "Line No": hdr = rec; continue
    if hdr is None or not rec[0]: continue
    if len(rec) < 8: continue
    try: s = int(rec[4])
    except ValueError: continue
    tot += s
    if cur != fname or not (l0 <= int(rec[0]) <= l1): continue
    st = {hdr[i][6:]: int(rec[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and rec[i].isdigit() and int(rec[i]) > 0}
    rows.append((int(rec[0]), s, int(rec[7]) if rec[7].isdigit() else 0, rec[1].strip()[:70], st))
print("total samples", tot)
for ln, s, ins, src, st in rows:
    if s == 0: continue
    top = ", ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
    print(f"{ln:5d} {100*s/tot:5.2f}% inst={ins:8d} | {src:70s} | {top}")
