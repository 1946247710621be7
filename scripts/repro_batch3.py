import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2509_10466_b200 import DsttConfig, DsttEngine, synth
cfg = DsttConfig.baseline(512, mask_dilate=5, mask_feather_sigma=3.0)
eng = DsttEngine(cfg, seed=0)
imgs, masks = synth.frame_pool("C5", 3)
rng = np.random.default_rng(0)
slots = [torch.from_numpy(rng.normal(0, 1, (3, cfg.tokens, 64)).astype(np.float32)).cuda() for _ in range(2)]
out_b, slot_b = eng.forward(torch.from_numpy(imgs).cuda(), torch.from_numpy(masks).cuda(), slots)
torch.cuda.synchronize(); print("ok")
