"""Per-region stall samples and executed instructions from an ncu report's source page.
Usage: python tools/ncu_hot.py report.ncu-rep [block]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
isrc, ie = hdr.index("Source"), hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
tots = sum(int(r[iss]) for r in data)
tot = sum(int(r[ie]) for r in data)
print(f"# {tot} warp instructions, {tots} stall samples")
KEY = ("LDG", "LDS", "STS", "BAR", "SYNCS", "ATOMS", "STG", "DADD", "CALL", "SHFL", "UBLKCP", "STL", "LDL")
for b in range(0, len(data), blk):
    part = data[b:b + blk]
    s = sum(int(r[iss]) for r in part)
    e = sum(int(r[ie]) for r in part)
    ops = [r[isrc].split()[1] if r[isrc].strip().startswith("@") else r[isrc].split()[0] for r in part]
    key = [o for o in ops if o.startswith(KEY)]
    top = max(part, key=lambda r: int(r[iss]))
    print(f"{b:4d}-{b + blk - 1:4d} samples {100 * s / tots:5.1f}% inst {100 * e / tot:5.1f}%  "
          f"{' '.join(key[:10])}  | top: {top[isrc].strip()[:48]} ({100 * int(top[iss]) / tots:.1f}%)")
