# quick per-step profile at 125M (1 step, tau=1)
import sys, time, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2411_02908_b200 import fedsim as F, _capi as A
m = F.ModelConfig(12, 768, 12, 4, 50368, 2048)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
corpus = F.generate_corpus("web", 2 * B * 2049 + 2049, 7, 50368)
plan = F.partition_iid(corpus, 1, 2048, 7)
t0 = time.time(); theta0 = F.TransformerModel(m).init_params(1); print("init", time.time()-t0, flush=True)
local = F.LocalTrainConfig(model=m, local_steps=1, batch_size=B)
r = F.FederationRunner(F.FederationConfig(1, 1, 5, 2, 42), local, F.ServerOptConfig(1, 0.1, 0.9, True), plan, theta0, precision="bf16")
for i in range(2):
    rec = r.run_round(); print("round", rec.round_ms, rec.local_ms, rec.aggregate_ms, rec.host_ms, rec.mean_client_loss, flush=True)
t = (C.c_double * 8)()
A.lib().photon_ctx_set_timing(r.ctx.handle, 1)
rec = r.run_round()
A.lib().photon_ctx_kernel_times(r.ctx.handle, t)
print("timed round", rec.round_ms, "gemm_ms %.2f attn_ms %.2f other_ms %.2f gemm TF/s %.1f launches %d" % (t[0], t[1], t[2], t[3]/t[0]/1e9, t[7]))
