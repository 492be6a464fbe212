"""Model load timing (profiling aid): AMNT file -> host tensors (load_model)
-> device handle (amun_model_create, incl. the tensor-core layouts)."""
import sys, time, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1610_01108_b200 import _lib, workload as W
from paper_1610_01108_b200.model import ModelConfig, load_model, random_model, save_model

cfg = ModelConfig(W.V_SRC, W.V_TRG, W.D_EMB, W.D_H, W.D_ATT)
with tempfile.TemporaryDirectory() as d:
    p = Path(d) / "m.amnt"
    save_model(random_model(cfg, 1), p)
    _lib.load()
    for it in range(3):
        t0 = time.perf_counter()
        m = load_model(p)
        t1 = time.perf_counter()
        dm = _lib.DeviceModel(m, 0)
        t2 = time.perf_counter()
        loader = getattr(_lib, "load_model_to_device", None)
        t3 = t2
        if loader:
            dm2 = loader(p, 0)
            t3 = time.perf_counter()
        print(f"load_model {1e3*(t1-t0):.0f} ms, amun_model_create {1e3*(t2-t1):.0f} ms"
              + (f", direct file->device {1e3*(t3-t2):.0f} ms" if loader else ""), flush=True)
        dm.close()
