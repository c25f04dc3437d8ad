"""Layout / cache-policy sweep on one generated configuration
(python tools/sweep.py --config cfg3 --policies 0,6 --stripes 0,1800000)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1402_3661_b200.corpus import _random_residue_limbs  # noqa: E402
from paper_1402_3661_b200.device import DeviceMatrix  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--policies", default="7")
    ap.add_argument("--stripes", default="0")
    ap.add_argument("--apw", default="0", help="comma list of SLD_APW_RATIO values; 0 = off")
    ap.add_argument("--chains", default="1", help="comma list of chains per matrix pass")
    ap.add_argument("--split", default="", help="comma list of SLD_SPLIT values (die split off/on)")
    ap.add_argument("--frac", default="", help="comma list of SLD_SPLIT_FRAC values")
    ap.add_argument("--bounds", default="", help="semicolon list of SLD_STRIPE_BOUNDS values")
    ap.add_argument("--pf", default="", help="comma list of SLD_PF values (index prefetch distance)")
    ap.add_argument("--envs", default="", help="semicolon list of K=V[,K=V] environment settings ('none' = none)")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    A, _, mod = bench.build_matrix(cfg, lambda m: print(m, file=sys.stderr))
    y = _random_residue_limbs(np.random.default_rng(5), A.total_cols, mod)
    splits = [(sp, fr, pf, bd, ev) for sp in (a.split.split(",") if a.split else [""])
              for fr in (a.frac.split(",") if a.frac else [""])
              for pf in (a.pf.split(",") if a.pf else [""])
              for bd in (a.bounds.split(";") if a.bounds else [""])
              for ev in (a.envs.split(";") if a.envs else ["none"])]
    extra_keys = set()
    for G, (sp, fr, pf, bd, ev) in [(int(x), s) for x in a.chains.split(",") for s in splits]:
      for k, val in (("SLD_SPLIT", sp), ("SLD_SPLIT_FRAC", fr), ("SLD_PF", pf), ("SLD_STRIPE_BOUNDS", bd)):
          if val:
              os.environ[k] = val
          else:
              os.environ.pop(k, None)
      for k in extra_keys:
          os.environ.pop(k, None)
      if ev and ev != "none":
          for kv in ev.split(","):
              k, v = kv.split("=", 1)
              os.environ[k] = v
              extra_keys.add(k)
      for sc in [int(x) for x in a.stripes.split(",")]:
        for pol, apw in [(int(x), float(y)) for x in a.policies.split(",") for y in a.apw.split(",")]:
            os.environ["SLD_POLICY"] = str(pol)
            if apw > 0:
                os.environ["SLD_APW"] = "1"
                os.environ["SLD_APW_RATIO"] = str(apw)
            else:
                os.environ.pop("SLD_APW", None)
            dm = DeviceMatrix(A, stripe_cols=sc, chains=G)
            v = dm.vector()
            v.upload_limbs(y if G == 1 else np.stack([y] * G))
            dm.bench(v, 10, 0)
            tot, per = dm.bench(v, a.steps, 0)
            tot2, per2 = dm.bench(v, a.steps, 0)
            per = min(per, per2)
            import subprocess
            clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu",
                                  "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
            inf = dm.info()
            print(f"{a.config} G={G} stripes={inf['stripes']} halves={inf['halves']} split_frac={fr or '-'} "
                  f"pf={pf or '-'} bounds={bd or '-'} env={ev} policy={pol} apw={apw}: "
                  f"{per:.4f} ms/pass = {per / G:.4f} ms per chain-product  [{clk}]",
                  flush=True)
            v.close()
            dm.close()


if __name__ == "__main__":
    main()
