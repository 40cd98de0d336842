import numpy as np, sys
t = np.load(sys.argv[1]).astype(np.int64)
t0 = t[:, 0].min()
r = lambda i: (t[:, i] - t0) / 1000.0
scan, lb, end, epi, st = r(4), r(5), r(6), r(3), r(2)
order = np.argsort(lb)
print("cta  stream  epi  scan  lookback  end   (lb-scan)")
for c in list(order[:5]) + list(order[-12:]):
    print(f"{c:4d} {st[c]:7.1f} {epi[c]:6.1f} {scan[c]:6.1f} {lb[c]:7.1f} {end[c]:6.1f}  {lb[c]-scan[c]:5.1f}")
print("max scan_start", scan.max(), "argmax", scan.argmax())
print("corr(lb-scan, cta index)", np.corrcoef(lb - scan, np.arange(len(lb)))[0, 1])
