"""One client step for profiling: a warm-up round then one round (tau=1).
  python tools/profile_step.py [B] [125m|1.3b]"""
import sys

sys.path.insert(0, "/root/repo")
from paper_2411_02908_b200 import _capi as A  # noqa: E402
from paper_2411_02908_b200 import fedsim as F  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shape = {"125m": (12, 768, 12, 4, 50368, 2048), "1.3b": (24, 2048, 16, 4, 50368, 2048)}[
    sys.argv[2] if len(sys.argv) > 2 else "125m"]
m = F.ModelConfig(*shape)
corpus = F.generate_corpus("web", 2 * B * 2049 + 2049, 7, 50368)
plan = F.partition_iid(corpus, 1, 2048, 7)
theta0 = F.TransformerModel(m).init_params(1)
local = F.LocalTrainConfig(model=m, local_steps=1, batch_size=B)
r = F.FederationRunner(F.FederationConfig(1, 1, 2, 2, 42), local, F.ServerOptConfig(1, 0.1, 0.9, True),
                       plan, theta0, precision="bf16")
for _ in range(2):
    n0 = A.lib().photon_launch_count()
    rec = r.run_round()
    print("round_ms", rec.round_ms, "loss", rec.mean_client_loss, "kernel launches",
          A.lib().photon_launch_count() - n0, flush=True)
