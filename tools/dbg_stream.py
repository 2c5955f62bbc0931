import json, sys, subprocess
sys.path.insert(0, "/root/repo")
import paper_2604_08812_b200 as d
w = json.load(open("/root/repo/tests/golden/wave.json"))
for exact in (True, False):
    with d.Engine(32, 16, 12, algorithm="left", storage=2) as eng:
        eng.load_kbf("/root/repo/tests/golden/wave.kbf", exact_columns=exact)
        eng.run()
        print("py stream exact", exact, [r["chosen_index"] for r in eng.trace()][:6], [round(r["gain"], 4) for r in eng.trace()][:3])
print("gold", w["chosen"][:6], [round(x, 4) for x in w["gains"][:3]])
r = subprocess.run(["/root/repo/paper_2604_08812_b200/lib/doptsel", "select", "/root/repo/tests/golden/wave.kbf", "--budget", "12", "--storage", "stream", "--out", "/tmp/o"], capture_output=True, text=True)
print(r.returncode, r.stderr, open("/tmp/o/trace.csv").read()[:300])
