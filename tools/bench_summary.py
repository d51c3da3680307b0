import json,sys
for line in sys.stdin:
    line=line.strip()
    if not line.startswith("{"): continue
    d=json.loads(line)
    print(d["config"]["workload"][:3], d["config"]["stream"], "%.3e traj-steps/s"%d["trajectory_steps_per_s"], "roof %.4f"%d["roofline"]["frac"], "e2e %.3e"%d["e2e"]["value"], d["config"]["engine"], d.get("clocks"))
