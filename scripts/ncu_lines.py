"""Top source lines of an ncu report (--import-source on, -lineinfo build):
python scripts/ncu_lines.py report.ncu-rep [top] [--sectors]
  default   : by warp-stall samples (with the two leading stall reasons)
  --sectors : by L2 theoretical global sectors (where the L2 traffic of the kernel comes from)"""
import collections, csv, io, subprocess, sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
by_sectors = "--sectors" in sys.argv
rep = args[0]
top = int(args[1]) if len(args) > 1 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, sec, src = collections.Counter(), collections.Counter(), {}
stall = collections.defaultdict(collections.Counter)
cur_file, cur, hdr = None, None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        i_s = hdr.index("Warp Stall Sampling (All Samples)")
        i_l2 = hdr.index("L2 Theoretical Sectors Global")
        cols = [j for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if r[0] != "":
        cur = (cur_file, int(r[0]))
        src[cur] = r[1].strip()[:80]
        continue
    try:
        agg[cur] += int(r[i_s] or 0)
        sec[cur] += int(float(r[i_l2] or 0))
        for j in cols:
            if r[j].isdigit():
                stall[cur][hdr[j]] += int(r[j])
    except (ValueError, IndexError):
        pass
key = sec if by_sectors else agg
tot = sum(key.values())
print(f"{rep}: {tot} {'L2 theoretical sectors' if by_sectors else 'warp-stall samples'}")
for (f, l), v in key.most_common(top):
    why = ", ".join(f"{k[6:]} {c * 100 // max(agg[(f, l)], 1)}%" for k, c in stall[(f, l)].most_common(2))
    print(f"{v / max(tot, 1) * 100:5.1f}%  {f}:{l:<5} {src.get((f, l), ''):80s}  [{why}]")
