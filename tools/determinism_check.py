"""Run the same short 125M federation twice (fresh runners, same seeds) and
compare per-round losses and theta bit for bit."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

from paper_2411_02908_b200 import fedsim as F  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tau = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m = F.ModelConfig(12, 768, 12, 4, 50368, 2048)
corpus = F.generate_corpus("web", 3 * tau * B * 2049 + 2049, 7, 50368)
plan = F.partition_iid(corpus, 1, 2048, 7)
theta0 = F.TransformerModel(m).init_params(1)
res = []
for trial in range(2):
    local = F.LocalTrainConfig(model=m, local_steps=tau, batch_size=B)
    r = F.FederationRunner(F.FederationConfig(1, 1, 3, 2, 42), local,
                           F.ServerOptConfig(1, 0.1, 0.9, True), plan, theta0, precision="bf16")
    losses = [r.run_round().mean_client_loss for _ in range(3)]
    th = r.theta()
    res.append((losses, th))
    print(f"trial {trial}: losses {losses}", flush=True)
    del r
same = res[0][1].tobytes() == res[1][1].tobytes()
print("theta identical:", same, " max|diff|", float(np.max(np.abs(res[0][1] - res[1][1]))))
