import os,sys; sys.path.insert(0,".")
import torch
from paper_2603_14371_b200.pi05 import Pi05Backend, Pi05Config, Pi05Observation, synthetic_images
be=Pi05Backend(Pi05Config(), num_blocks=64)
for i in range(3):
    kv=be.prefill(Pi05Observation(tuple(range(100,132)),0,synthetic_images(3,5))); torch.cuda.synchronize(); print("prefill ok", i, flush=True)
    del kv
