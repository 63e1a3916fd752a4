import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import json
from golden_runner import run_case
from paper_2604_07311_b200.engine import _lib
for opt in sys.argv[2:]:
    k, v = opt.split("=")
    _lib.lib().bf_set_option(k.encode(), int(v))
g = json.load(open("tests/golden/golden.json"))
c = [x for x in g["cases"] if x["id"] == sys.argv[1]][0]
outs, err = run_case(c, "cuda")
from golden_inputs import digest
print("ok", err, digest(list(outs.values())[0]) == list(c[list(outs)[0]].values())[0] if False else "", flush=True)
print("match", digest(outs["a_out"]) == c["a_out"]["sha256"])
