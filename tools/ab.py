"""A/B timing of alternative libsgad builds on the same box:
python tools/ab.py variants/a.so variants/b.so ..."""
import json, os, subprocess, sys
for lib in sys.argv[1:]:
    env = dict(os.environ, SGAD_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "2", "--no-cpu-baseline",
                          "--no-e2e", "--no-track"], capture_output=True, text=True, env=env)
    for l in out.stdout.splitlines():
        if l.startswith("{"):
            d = json.loads(l); r = d["roofline"]
            f = lambda k: "   -  " if r.get(k) is None else f"{r[k]:.3f}"
            print(f"{lib:30s} step {d['ms_per_step']:.2f} ms  prep {r['prepare_ms_per_view']:.3f}  "
                  f"fwd {f('forward_ms_per_view')}  bwd {f('backward_ms_per_view')}  "
                  f"fb {f('forward_backward_ms_per_view')}", flush=True)
    if out.returncode:
        print(lib, "failed", out.stderr[-500:])
