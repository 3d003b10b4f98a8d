"""Print condense/step times of the exp_env.sh A/B logs."""
import glob
import json
for f in sorted(glob.glob("gpurun_out/exp_*.log")):
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
            print(f"{f:36s} condense {d['condense_ms']:8.2f} ms  step {d['ms_per_step']:8.2f} ms  frac {d['roofline']['frac']:.3f}")
            break
    else:
        print(f, "FAILED:", open(f).read()[-300:])
