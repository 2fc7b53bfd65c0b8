import json, os, sys
import numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import rel_err
from paper_2507_05753_b200 import Communicator, ModelConfig, MpContext, WeatherMixerModel
z = np.load("tests/golden/wm_golden.npz"); meta = json.load(open("tests/golden/comm_golden.json"))
for dtype in sys.argv[1:] or ["f32"]:
    m = WeatherMixerModel(MpContext(Communicator.local(), [0]), ModelConfig.from_dict(meta["config"]), dtype=dtype)
    m.zero_grads()
    out = m.forward(torch.tensor(z["x"], dtype=torch.float32))
    m.backward(torch.tensor(z["g_out"], dtype=torch.float32))
    torch.cuda.synchronize()
    print(dtype, "out", rel_err(out.cpu().numpy(), z["out_f64"]))
    for name in meta["param_names"]:
        g = m.params[name].grad.cpu().numpy(); r = z["grad_f64/" + name]
        print(f"  {name:18s} {rel_err(g, r):.2e}  |g| {np.abs(g).max():.3e} |ref| {np.abs(r).max():.3e}")
