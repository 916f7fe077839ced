"""Memory-stability check: 4 rounds of 100 streamed + 50 sequential config-0 maps;
GPU memory in use and host max RSS must stay flat (pools recycle)."""
import numpy as np, torch, resource
import paper_2403_07631_b200 as pct
from paper_2403_07631_b200 import synth, _lib
from paper_2403_07631_b200.batch import BatchRunner, stream_maps
xyz = synth.generate(0)
run = BatchRunner(0, workers=2)
def mem():
    f, t = torch.cuda.mem_get_info(0)
    return (t - f) / 2**20, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024
for rnd in range(4):
    for t in stream_maps([xyz] * 100, 0.5, 0.1, pct.TravParams(), runner=run):
        pass
    for _ in range(50):
        tom = pct.simplify_tomogram(pct.evaluate_tomogram(pct.build_tomogram(pct.PointCloud(xyz), 0.5, 0.1), pct.TravParams())).materialize()
    print(rnd, "gpu MiB used %.0f, host maxrss MiB %.0f" % mem())
