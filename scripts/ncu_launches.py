"""One eager (un-captured) full inference, bracketed by cudaProfilerStart/Stop, so that
`ncu --profile-from-start off --metrics gpu__time_duration.sum` lists exactly the kernels of one
inference (weight generation and warm-up are outside the profiled range).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python scripts/ncu_launches.py [views] [prompt]
"""
import ctypes
import os
import sys

# the production (clustered) megakernel without the cooperative attribute, which ncu cannot replay
os.environ.setdefault("PI0B_AE_COOP", "0")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = default_config(views=views, prompt_tokens=prompt)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
x = gen_inputs(cfg, 1)
eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))  # warm-up (module load, first-touch)
drv = ctypes.CDLL("libcuda.so.1")  # the engine's (primary) context is current on this thread
drv.cuProfilerStart()
eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
drv.cuProfilerStop()
print("kernels per inference:", eng.kernel_count(0))
