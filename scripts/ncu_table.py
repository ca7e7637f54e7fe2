"""Dev tool: per-kernel table from an `ncu --metrics ... --csv` log."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data.setdefault((int(d["ID"]), d["Kernel Name"][:48]), {})[d["Metric Name"]] = d["Metric Value"]
    print("==", path)
    for (i, k), m in data.items():
        print(f"{i:3d} {k:48s} " + " ".join(f"{n.split('__')[1][:14]}={v}" for n, v in m.items()))
