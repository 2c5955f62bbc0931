import json, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2604_08812_b200 as d
from oracle import oracle as O
cases = json.load(open("/root/repo/tests/golden/random.json"))["cases"]
for ci, c in enumerate(cases):
    nd, nt = c["n_sensors"], c["n_steps"]
    k = O.random_hessian(nd, nt, c["gamma"], c["rank"], c["seed"])
    eng = d.Engine(nd, nt, c["budget"], algorithm="left")
    eng.load_k(k)
    eng.run()
    rows = eng.trace()
    eng.close()
    got = [r["chosen_index"] for r in rows]
    bad = [i for i, (r, g) in enumerate(zip(rows, c["gains"])) if abs(r["gain"] - g) > 1e-9 * max(abs(g), 1)]
    print(ci, nd, nt, c["budget"], "seq ok" if got == c["chosen"] else f"seq {got} vs {c['chosen']}", "bad rounds", bad[:5])
