"""Small selections for compute-sanitizer (racecheck / synccheck / memcheck):
every round kernel of each algorithm and storage variant runs at least once
(nt = 32: triangle-resident gain kernel; 130: panel gain kernel; 3: odd-nt
update path).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_08812_b200 as d  # noqa: E402

for (nd, nt, rank, b) in [(24, 32, 256, 4), (6, 130, 600, 3), (10, 3, 20, 4)]:
    v = d.synthetic_v(nd, nt, rank, 2024)
    seqs = []
    for kw in (dict(), dict(packed=False), dict(algorithm="left"), dict(algorithm="left", storage="stream")):
        with d.Engine(nd, nt, b, export_factor=True, **kw) as eng:
            eng.gen_synthetic(v, rank, 1.0)
            eng.run()
            seqs.append([r["chosen_index"] for r in eng.trace()])
            eng.export_factor(b)
    assert all(s == seqs[0] for s in seqs), seqs
    print("sanitize_run ok", nd, nt, seqs[0], flush=True)
