"""Times device-side generation (sfseg_synth_generate_device) of a BASELINE
config against the host generator on a T-cropped sample.
usage: python tools/time_synth.py [--config 4] [--host-frames 8]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1907_02731_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--host-frames", type=int, default=8)
args = ap.parse_args()

prob = synth.config(args.config)[0]
T, H, W = prob.shape
fields = 1 + prob.channels
prob.generate_device()  # warm-up (jump table, module load)
torch.cuda.synchronize()
t0 = time.perf_counter()
S, F, _ = prob.generate_device()
torch.cuda.synchronize()
dev_s = time.perf_counter() - t0
bytes_ = fields * prob.voxels() * 4
del S, F
hp = synth.config(args.config, frames=args.host_frames)[0]
t0 = time.perf_counter()
hp.generate()
host_s = (time.perf_counter() - t0) * T / args.host_frames
print(json.dumps({"config": f"c{args.config}", "shape": [T, H, W], "fields": fields,
                  "device_s": dev_s, "device_GBps": bytes_ / dev_s / 1e9,
                  "host_s_extrapolated": host_s, "host_threads": os.cpu_count(),
                  "host_sample_frames": args.host_frames}))
