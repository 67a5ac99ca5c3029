"""Two federated rounds of a small bf16 / f32 model through the library
PHOTON_LIB names; theta written to argv[1] (bitwise A/B of two builds)."""
import sys

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402

from paper_2411_02908_b200 import fedsim as F  # noqa: E402

prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
shape = (2, 256, 4, 4, 96, 160)  # dh = 64: tcgen05 attention, fused dh-64 backward
m = F.ModelConfig(*shape)
corpus = F.generate_corpus("web", 200000, 7, 96)
plan = F.partition_iid(corpus, 2, 160, 7)
theta0 = F.TransformerModel(m).init_params(1)
local = F.LocalTrainConfig(model=m, local_steps=3, batch_size=4)
r = F.FederationRunner(F.FederationConfig(2, 2, 2, F.Topology.kRingAllReduce, 42), local,
                       F.ServerOptConfig(1, 0.1, 0.9, True), plan, theta0, precision=prec)
for _ in range(2):
    print(r.run_round().mean_client_loss)
np.save(sys.argv[1], r.theta())
