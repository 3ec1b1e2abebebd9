"""Hash of device f+grad outputs (fused and partial paths) at c1-c3 shapes: bitwise A/B of two builds
(MCP_LIBRARY=<other .so> python tools/hash_outputs.py)."""
import hashlib, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1911_03813_b200 as mcp
from paper_1911_03813_b200 import synth, _native
h = hashlib.sha256()
for name, p in (("c1", None), ("c2", 200000), ("c3", 50000)):
    cfg = synth.CONFIGS[name]
    V = synth.device_observations(cfg, 7, p=p)
    obs = mcp.ObservationSet.from_device(V, p_total=V.shape[0])
    ctx = obs.device_context()
    lam, A = synth.initial_point(cfg, 7)
    x = torch.as_tensor(mcp.pack(lam, A), device="cuda")
    out = torch.empty(1 + cfg.r + cfg.n * cfg.r, dtype=torch.float64, device="cuda")
    s = _native.stream_handle(torch.cuda.current_stream())
    ctx.fg_device(cfg.d, cfg.r, x.data_ptr(), 0.3, None, out.data_ptr(), s)
    Yw = torch.empty(cfg.n * cfg.r + cfg.r, dtype=torch.float64, device="cuda")
    ctx.fg_partial_device(cfg.d, cfg.r, x.data_ptr(), None, Yw.data_ptr(), s)
    torch.cuda.synchronize()
    h.update(out.cpu().numpy().tobytes()); h.update(Yw.cpu().numpy().tobytes())
    print(name, ctx.last_variant)
print("HASH", h.hexdigest())
