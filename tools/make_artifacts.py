"""Build (or load) the setup artifacts of a configuration with the product's
own setup path (KL basis: LAPACK/ARPACK via scipy; k-means: GPU distance
sweeps + host means) and copy them to gpurun_out/artifacts/ so a gpurun call
can bring them back into this container's artifacts/ cache."""
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_07824_b200 import campaign  # noqa: E402

names = sys.argv[1:] or ["C1", "C2", "C3", "C5"]
out = os.path.join(campaign.ROOT, "gpurun_out", "artifacts")
os.makedirs(out, exist_ok=True)
for name in names:
    cfg = campaign.CONFIGS[name]
    t = time.time()
    arts = campaign.prepare_campaign(cfg)
    print(name, "basis", arts["basis"]["eigenvalues"].size, "P", arts["codebook"]["P"], f"{time.time() - t:.1f}s",
          flush=True)
keep = set()
for name in names:  # only the requested configurations' files (gpurun brings back <= 64 MiB)
    cfg = campaign.CONFIGS[name]
    keep.add(f"basis_{campaign._key(cfg, 'basis')}.klb")
    keep.add(f"codebook_{campaign._key(cfg, 'codebook')}.qnt")
for f in sorted(keep):
    if os.path.exists(os.path.join(campaign.CACHE, f)):
        shutil.copy(os.path.join(campaign.CACHE, f), out)
print("copied", os.listdir(out))
