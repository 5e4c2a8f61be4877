"""Which problems of a config diverge on the device (FAST and STRICT)?"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1108_1688_b200 as hj
from paper_1108_1688_b200 import workloads as W
cfg = int(sys.argv[1]); modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fast", "strict"]
probs = W.make_config(cfg)
for mode in modes:
    s = hj.Solver(probs, mode=mode)
    try:
        s.run()
    except hj.api.HjmsvError as e:
        print(mode, "error:", e)
    bad = [(q, s.report(q)["status"], s.report(q)["failed_step"]) for q in range(len(probs)) if s.report(q)["status"]]
    print(mode, "failed problems:", bad)
    s.close()
