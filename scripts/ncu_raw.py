"""Print selected raw metrics of every kernel in an .ncu-rep (name: value unit)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
mets = sys.argv[2].split(",")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:60])
    for m in mets:
        if m in hdr:
            i = hdr.index(m)
            print(f"   {m:70s} {r[i]} {units[i]}")
