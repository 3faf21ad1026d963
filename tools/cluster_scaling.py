"""C2 throughput vs the number of resident clusters (FKS_MAX_CLUSTERS), development aid."""
import os, subprocess, sys
for m in [4, 8, 15, 18]:
    env = dict(os.environ, FKS_MAX_CLUSTERS=str(m))
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "quick_time.py")], env=env,
                         capture_output=True, text=True).stdout
    c2 = [l for l in out.splitlines() if l.startswith("C2")]
    print(m, "clusters:", c2[0] if c2 else out[-300:], flush=True)
