"""Fill DESIGN.md's @@...@@ result placeholders from a capture directory: python tools/fill_design.py profiles/r02y"""
import json
import re
import sys

d = sys.argv[1].rstrip("/")
tag = d.split("/")[-1]
j = lambda n: json.load(open(f"{d}/bench_{n}.json"))
c5, c4, g2 = j("c5"), j("c4"), j("c4_gloo2")
M = lambda v: f"{v / 1e6:.1f} M"
r5, r4 = c5["roofline"], c4["roofline"]
ntests = re.search(r"(\d+) passed", open(f"{d}/pytest_gpu.log").read()).group(1)
rep = {
    "FINAL": tag, "NTESTS": ntests,
    "C5": M(c5["value"]), "C5RAYS": M(c5["rays_per_s"]["device"]), "C5E2E": M(c5["e2e"]["value"]),
    "C5FRAC": f"{100 * r5['frac']:.1f} %", "C5SHARE": f"{100 * r5['kernel_share']:.0f} %",
    "C5LSHARE": f"{100 * r5['step']['k_wf_logic_share']:.0f} %",
    "C5CEIL": f"{100 * r5['traversal_ceiling']['frac']:.0f} %",
    "REL": f"{c5['relmse']['ratio']:.3f}", "ACC": f"{c5['acceptance']['value']:.3f}",
    "C4": M(c4["value"]), "C4E2E": M(c4["e2e"]["value"]), "C4FRAC": f"{100 * r4['frac']:.1f} %",
    "C4SHARE": f"{100 * r4['kernel_share']:.0f} %",
    "G2": M(g2["value"]), "G2E2E": M(g2["e2e"]["value"]), "G2ACC": f"{g2['acceptance']['value']:.3f}",
}
s = open("DESIGN.md").read()
for k, v in rep.items():
    s = s.replace(f"@@{k}@@", v)
open("DESIGN.md", "w").write(s)
print("left:", sorted(set(re.findall(r"@@\w+@@", s))))
