"""Parameter sweep (dev helper): env knobs x configs -> run stats."""
import itertools, json, os, subprocess, sys
cfgs = [int(x) for x in sys.argv[1].split(",")]
knobs = json.loads(sys.argv[2])  # {"GP_DELTA_FACTOR": ["inf","4"], ...}
keys = list(knobs)
for vals in itertools.product(*[knobs[k] for k in keys]):
    env = dict(os.environ, **dict(zip(keys, vals)))
    for c in cfgs:
        out = subprocess.run([sys.executable, "scripts/quick_run.py", str(c)], env=env,
                             capture_output=True, text=True, timeout=900)
        last = [l for l in out.stdout.splitlines() if "rep1" in l]
        print(dict(zip(keys, vals)), last[-1] if last else out.stderr[-500:], flush=True)
