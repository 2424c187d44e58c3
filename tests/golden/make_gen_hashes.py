"""Records the device checksums of the seeded BASELINE matrices (paper_2502_19284_b200/gen.py) as
tests/golden/gen_hashes.json.  Run on a B200 box (the torch CUDA generator is the RNG):
    python tests/golden/make_gen_hashes.py [configs...]
tests/test_gpu_gen.py regenerates each matrix and compares against these numbers, so the two bench
arms (separate processes) and every test see bit-identical inputs."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

from gen_checksum import checksum  # noqa: E402
from paper_2502_19284_b200 import gen  # noqa: E402

out = os.path.join(HERE, "gen_hashes.json")
cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
data = json.load(open(out)) if os.path.exists(out) else {}
for k in cfgs:
    name, fn = gen.CONFIGS[k]
    m, n, r, c, v = fn("cuda")
    data[str(k)] = {"name": name, "m": m, "n": n, "nnz": int(v.numel()), "checksum": checksum(r, c, v),
                    "torch": torch.__version__, "device": torch.cuda.get_device_name()}
    print(k, data[str(k)], flush=True)
    del r, c, v
    torch.cuda.empty_cache()
json.dump(data, open(out, "w"), indent=1)
