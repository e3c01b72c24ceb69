import sys
sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs
wl = configs.make(sys.argv[1]); eng = Engine(0); k = Kernel.parse(wl.kernel)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0); p = ParticleSet(wl.xyz, wl.weights)
eng.cstc_sum(p, p, k, cfg, SumStats())
