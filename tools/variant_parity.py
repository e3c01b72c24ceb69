"""Developer probe: full-size parity of library variants against the reference.

python tools/variant_parity.py c5 [c3 c2 ...]  — for each config, the reference's csfmm_sum
(oracle/_ref, host cores) is computed once and cached under /tmp; then every
_variants/*/libcsfs_b200.so (and the in-tree library) is run in a subprocess
(CSFS_B200_LIB) and its relative L2 against the reference printed (one JSON line per
variant and config)."""
import glob
import json
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, ".")


def child(name, out):
    from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs

    wl = configs.make(name)
    eng = Engine(0)
    st = SumStats()
    p = ParticleSet(wl.xyz, wl.weights)
    g = eng.csfmm_sum(p, p, Kernel.parse(wl.kernel), TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0),
                      st).values
    np.save(out, g)


def main():
    if sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        return
    from oracle import ref
    from paper_2508_13550_b200 import configs

    os.makedirs("gpurun_out", exist_ok=True)
    libs = sorted(glob.glob("_variants/*/libcsfs_b200.so")) + ["paper_2508_13550_b200/libcsfs_b200.so"]
    for name in sys.argv[1:]:
        cache = f"/tmp/ref_{name}.npy"
        if not os.path.exists(cache):
            wl = configs.make(name)
            r, _ = ref.csfmm(wl.xyz, wl.xyz, wl.weights, wl.kernel, mac=wl.mac, degree=wl.degree, n0=wl.n0)
            np.save(cache, r)
        r = np.load(cache)
        for lib in libs:
            out = "/tmp/variant_out.npy"
            env = dict(os.environ, CSFS_B200_LIB=os.path.abspath(lib))
            subprocess.run([sys.executable, __file__, "--child", name, out], env=env, check=True)
            g = np.load(out)
            e = float(np.sqrt(np.sum((g - r) ** 2) / np.sum(r ** 2)))
            m = float(np.max(np.abs(g - r)) / np.max(np.abs(r)))
            print(json.dumps({"cfg": name, "lib": lib, "rel_l2": e, "max_rel": m}), flush=True)


if __name__ == "__main__":
    main()
