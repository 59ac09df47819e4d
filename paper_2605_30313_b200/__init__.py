"""B200-native UniLab learner hot path (drop-in for the reference ``unilite``
learner API).  Compute runs in libunilite_b200.so (sm_100a); PyTorch is the
host shell for HBM allocations, streams and torch.distributed."""

__version__ = "0.1.0"
