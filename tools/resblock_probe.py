"""Per-launch device times of one OTSM ResBlock (720p level-0 shape by default) for same-box
experiments: shift ratio, widths, engine knobs (DVC_LIB / DVC_* in experiment builds).
    python tools/resblock_probe.py [--cin 240] [--cout 240] [--h 90] [--w 160] [--T 32] [--p 8]"""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2601_20564_b200 as dvc  # noqa: E402
import synthgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cin", type=int, default=240)
ap.add_argument("--cout", type=int, default=240)
ap.add_argument("--h", type=int, default=90)
ap.add_argument("--w", type=int, default=160)
ap.add_argument("--T", type=int, default=32)
ap.add_argument("--p", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dt = torch.bfloat16
wt = {k: (None if v is None else torch.from_numpy(v).to(dt).cuda())
      for k, v in synthgen.resblock_weights(a.cin, a.cout).items()}
prm = dvc.ResBlockParams(wt, a.cin, 0, 24, a.p)
x = torch.from_numpy(synthgen.normal((a.T, a.h, a.w, a.cin), 3)).to(dt).cuda()
carry = torch.from_numpy(synthgen.normal((a.h, a.w, a.cin), 4)).to(dt).cuda() if a.p else None
out = torch.empty((a.T, a.h, a.w, a.cout), dtype=dt, device="cuda")
ws = torch.empty(prm.workspace_size(a.T, a.h, a.w), dtype=torch.uint8, device="cuda")
run = lambda: dvc.dvc_resblock_tsm_forward(prm, x, carry_in=carry, out=out, workspace=ws)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
acc = collections.OrderedDict()
for _ in range(a.reps):
    dvc.profile_begin(256)
    run()
    dvc.profile_end()
    for lab, ms, fl in dvc.profile_records():
        e = acc.setdefault(lab, [0.0, fl, 0])
        e[0] += ms
        e[2] += 1
for lab, (ms, fl, n) in acc.items():
    t = ms / n
    print(f"{lab:50s} {t * 1e3:8.1f} us" + (f"  {fl / t / 1e9:7.1f} TF/s" if fl else ""))
