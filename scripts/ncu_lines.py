"""Top source lines by warp-stall samples from an ncu report (--import-source on):
python scripts/ncu_lines.py report.ncu-rep [top]"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, src, stall = collections.Counter(), {}, collections.defaultdict(collections.Counter)
cur_file, cur, hdr = None, None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if r[0] != "":
        cur = (cur_file, int(r[0]))
        src[cur] = r[1].strip()[:80]
        continue
    try:
        agg[cur] += int(r[i_s])
        for j in cols:
            if r[j].isdigit():
                stall[cur][hdr[j]] += int(r[j])
    except (ValueError, IndexError):
        pass
tot = sum(agg.values())
print(f"{rep}: {tot} warp-stall samples")
for (f, l), v in agg.most_common(top):
    why = ", ".join(f"{k[6:]} {c * 100 // max(v, 1)}%" for k, c in stall[(f, l)].most_common(2))
    print(f"{v / tot * 100:5.1f}%  {f}:{l:<5} {src.get((f, l), ''):80s}  [{why}]")
