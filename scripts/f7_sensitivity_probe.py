"""Sensitivity of one pixel's oracle radiance to tiny turns of its primary ray (16 directions x 6 scales).
Development aid behind the three-scale F7 (reading 22); edit the pixel below."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1702_01530_b200 import scenes
from oracle.oracle import Oracle
s = scenes.scene_c3()
O = Oracle(s)
cam = O.camera()
o, d = O.primary_ray(cam, 0, 1750, 601)
base = np.clip(O.trace_ray(o, d, s.max_depth)[0], 0, 1)
a = np.array([1.0, 0, 0])
u = np.cross(d, a); u /= np.linalg.norm(u); w = np.cross(d, u)
for ang in np.linspace(0, 2*np.pi, 16, endpoint=False):
    q = np.cos(ang) * u + np.sin(ang) * w
    row = []
    for eps in (2e-8, 5e-8, 1e-7, 2e-7, 5e-7, 1e-6):
        dd = d + eps * q; dd /= np.linalg.norm(dd)
        r = np.clip(O.trace_ray(o, dd, s.max_depth)[0], 0, 1)
        row.append(np.abs(r - base).max())
    print(f"{ang:5.2f}", " ".join(f"{x:8.1e}" for x in row))
