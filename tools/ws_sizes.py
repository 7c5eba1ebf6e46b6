import sys; sys.path.insert(0,'.')
import torch, ctm_inputs as ci
from paper_2306_08212_b200 import ctm
for name in ["c4","c5","c5_256"]:
    cfg=ci.CONFIGS[name]
    for flags,lab in [(ctm.CTM_FLAG_MOVE_ONLY,"move_only"),(0,"all")]:
        h=ctm.CtmHandle(cfg.d,cfg.D,cfg.chi,cfg.chi_p,cfg.chi_pp,flags=flags)
        print(name, lab, "ws GB", h.ws_bytes/1e9, flush=True)
        del h; torch.cuda.empty_cache()
