"""Print ncu --csv (long format) metrics side by side per kernel launch."""
import csv, sys, collections
for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    rows = rows[[i for i, r in enumerate(rows) if "Kernel Name" in r][0]:]
    h = rows[0]; ki = h.index("Kernel Name"); mi = h.index("Metric Name"); vi = h.index("Metric Value"); ii = h.index("ID")
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault((r[ii], r[ki][:45]), {})[r[mi]] = r[vi]
    print("==", f)
    for (i, k), m in d.items():
        print(i, k, " ".join(f"{n.split('__')[1][:22]}={v}" for n, v in m.items()))
