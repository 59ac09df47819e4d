import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import test_gpu_ppo as T
import paper_2605_30313_b200 as P
from paper_2605_30313_b200 import algos as A, tensornet as TN
P.set_precision("fp32")
mode = sys.argv[1] if len(sys.argv) > 1 else "both"
if mode in ("both", "pre"):
    T.test_learners_and_weight_slot()
def run():
    prec = "fp32"
    T_, N = 8, 512
    segs = []
    for sd in (3, 4, 5):
        segd, actor, critic = T._synthetic(T_, N, 48, 52, 12, (128, 64), seed=sd)
        segs.append(A.RolloutSegment(**segd))
    cfg = A.PpoConfig(epochs=2, minibatches=2)
    arch_a, arch_c = TN.Arch(48, (128, 64), 12), TN.Arch(52, (128, 64), 1)
    def fresh():
        p = A.AcParams(TN.ModelParams.from_numpy(arch_a, actor.flat()),
                       TN.ModelParams.from_numpy(arch_c, critic.flat()))
        return p, A.AcOpt.for_params(p, cfg.lr)
    p1, o1 = fresh()
    rng1 = A.DeviceRng(7)
    serial = []
    for sg in segs:
        sg.advantages, sg.returns = A.gae(sg.rewards, sg.values, sg.terminated, sg.truncated,
                                          sg.bootstrap_value, cfg.gamma, cfg.lam,
                                          truncation_values=sg.truncation_values)
        serial.append(A.ppo_update(sg, p1, o1, cfg, rng1))
    p2, o2 = fresh()
    pipe = A.PpoPipeline(p2, o2, cfg, A.DeviceRng(7))
    pipe.prefetch(segs[0])
    piped = []
    for i in range(len(segs)):
        piped.append(pipe.update(next_segment=segs[i + 1] if i + 1 < len(segs) else None))
    return [(round(a.policy_loss, 6), round(b.policy_loss, 6)) for a, b in zip(serial, piped)]
for it in range(6):
    print(it, run(), flush=True)
