import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2505_18231_b200 as P
from tests.conftest import codebook_for, load_golden
from tests.golden.inputs import pipeline_inputs
for case in pipeline_inputs():
    g = load_golden(f"pipeline_{case['name']}.npz")
    cb = codebook_for(case["bit_mode"])
    res = []
    for prec in ("precise", "balanced", "fast"):
        cfg = P.CacheConfig(d=128, bit_mode=cb.bit_mode, strategy=P.ScaleStrategy(case["strategy"]))
        c = P.PagedKvCache(cfg, 1, 1, cb_k=cb, cb_v=cb, base_position=case["base_position"], precision=prec)
        K, V = case["keys"], case["values_ht"]
        import torch
        for a, b in case["batches"]:
            c.append(torch.from_numpy(K[a:b][None, None]).cuda(), torch.from_numpy(V[a:b][None, None]).cuda())
        out = c.attend(torch.from_numpy(case["q"][None]).cuda()).cpu().numpy()[0]
        err = max(np.max(np.abs(out[i] - g["out"][i])) / np.max(np.abs(g["out"][i])) for i in range(len(case["q"])))
        res.append(f"{prec} {err:.2e}")
    print(case["name"], " | ".join(res))
