import faulthandler, sys, time, os
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(40, exit=True)
import torch
from paper_2004_09910_b200 import Pipeline, TgpError
from synth import configs as C
opts = dict(a.split("=") for a in sys.argv[1:])
layers = C.resmlp_stack(4, 256, hidden=512)
B, m = 32, 4
P = Pipeline(layers, chunks=m, devices=[0, 0], balance=[2, 2], checkpoint="except_last", max_batch=B, dtype="bf16", seed=3)
P.init_params(3)
for k, v in opts.items():
    P.set_option(k, int(v))
X = torch.randn(B, 256, device="cuda"); Y = torch.empty(B, 256, device="cuda")
print("fwd start", opts, flush=True); t0 = time.time()
try:
    P.forward(X, B, Y)
    print("fwd ok", time.time() - t0, flush=True)
except TgpError as e:
    print("raised", e.rc, e, time.time() - t0, flush=True)
P.close()
print("closed", flush=True)
