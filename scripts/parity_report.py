"""Large-sample parity report (test infrastructure; complements tests/test_gpu_parity.py).

Full-size frames of C3, C4 and C5 (frames 0 and 30) rendered in the bench's launch
configuration through the C ABI; the double-precision brute-force oracle evaluates a large
seeded pixel sample of each, and the north-star criteria are computed exactly as the tests do
(tests/parity.py): primary IDs bit-exact off the fragile set, RGB within 2/255 on >= 99.9 % of
pixels, max |radiance error| <= 1e-3 off the fragile set.
usage: python scripts/parity_report.py [n_per_eye] > profiles/<tag>_parity_report.json
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from oracle.oracle import Oracle  # noqa: E402
from paper_1702_01530_b200 import rt, scenes  # noqa: E402
from tests.parity import compare  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    R = rt.StereoRenderer(0)
    out = {}
    cases = [("C3", scenes.scene_c3(), 4 * n, 101), ("C4", scenes.scene_c4(), n, 102),
             ("C5 frame 0", scenes.scene_c5(frame=0), n // 2, 103), ("C5 frame 30", scenes.scene_c5(frame=30), n // 2, 104)]
    for label, s, per_eye, seed in cases:
        R.upload(s)
        R.set_camera(s.rig)
        g = R.render(s.width, s.height, s.max_depth, want_id=True, want_radiance=True)
        torch.cuda.synchronize()
        g = {k: v.cpu().numpy() for k, v in g.items()}
        pix = scenes.sample_pixels(s.width, s.height, per_eye, seed)
        t0 = time.time()
        ref = Oracle(s).render(pixels=pix)
        dt = time.time() - t0
        e, x, y = pix[:, 0], pix[:, 1], pix[:, 2]
        st = compare(ref, g["id"][e, y, x], g["fb"][e, y, x], g["radiance"][e, y, x], label)
        st.update({"width": s.width, "height": s.height, "max_depth": s.max_depth, "pixels_sampled": int(len(pix)),
                   "oracle_s": dt,
                   "pass": bool(st["id_mismatch"] == 0 and st["rgb_frac"] >= 0.999 and st["max_err"] <= 1e-3)})
        print(label, st, file=sys.stderr, flush=True)
        out[label] = st
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
