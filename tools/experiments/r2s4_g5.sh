# column-pair boxes: every ksg entry forced on n = 54 / 66 / 78 (what should the cost model pick?)
O=gpurun_out/s4g5
mkdir -p $O
python - > $O/sweep.log 2>&1 <<'PY'
import os, sys, json, subprocess
sys.path.insert(0, os.getcwd())
from paper_2208_09822_b200 import iaat
cat = [e for e in iaat.iaat_catalog_describe() if e["family"] == "ksg"]
for n in (42, 54, 66, 78):
    for tr in ("NN", "NT", "TT"):
        res = []
        for e in [None] + [e for e in cat if e["trans"] == tr]:
            env = dict(os.environ)
            if e is not None:
                env["IAAT_FORCE_FAMILY"] = "7"; env["IAAT_FORCE_ORDER"] = str(e["index"])
            r = subprocess.run([sys.executable, "tools/run_case.py", "f32", tr, str(n), str(n), str(n), "--reps", "6", "--plan"],
                               env=env, capture_output=True, text=True, timeout=120)
            out = r.stdout.strip().splitlines()
            us = None
            for l in out:
                if " us," in l: us = float(l.split(":")[1].split("us")[0])
            plan = out[0] if out else ""
            ent = e["index"] if e else -1
            tag = "" if e is None else "%dx%d l%d k%d u%d g%dw%d" % (e["mr"], e["nr"], e["lr"], e["kc"], e["ku"], e["g"], e["w"])
            import re
            m = re.search(r"'entry': (\d+).*'P': (\d+), 'S': (\d+)", plan)
            print(n, tr, ent, tag, us, m.groups() if m else r.stderr[-200:], flush=True)
PY
cat $O/sweep.log
