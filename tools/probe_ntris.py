import sys; sys.path.insert(0,'tools'); sys.argv=['x']
import probe
for n in (1<<10, 1<<14, 1<<17, 1<<20):
    probe.probe_c4(n_tris=n)
