"""Per-source-line hot spots from an ncu report (--import-source, -lineinfo):
python tools/ncu_lines.py report.ncu-rep [top]  -> warp-stall samples and executed instructions per line"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
files, out, hdr, fname = {}, [], None, "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit() and r[0] != "0":
        d = dict(zip(hdr[4:], r[4:]))
        try:
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        stalls = {h.replace("stall_", ""): int(r[i]) for i, h in enumerate(hdr)
                  if h.startswith("stall_") and "Not Issued" not in h and r[i].isdigit()}
        out.append((samp, inst, f"{fname}:{r[0]}", r[1].strip()[:70], stalls))
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"# {rep}: {tot_s} stall samples, {tot_i:.3e} warp instructions")
print(f"{'samp%':>6} {'inst%':>6}  {'line':18s} top stalls | source")
for samp, inst, loc, src, st in sorted(out, reverse=True)[:top]:
    ts = ",".join(f"{k}:{v * 100 // max(samp, 1)}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{100 * samp / tot_s:6.2f} {100 * inst / tot_i:6.2f}  {loc:18s} {ts:40s} | {src}")
