"""Files written by the REFERENCE dataio (dataio.py) for the format tests.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_io.py

Writes tests/golden/io/{points.fcpt, points.csv, sdf.ckpt, cams.json,
img.ppm} and io.npz (the arrays they hold, as the reference loads them).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fc2t2 import dataio  # noqa: E402
from fc2t2.ray import Camera  # noqa: E402

OUT = Path(__file__).resolve().parent / "io"


def main():
    OUT.mkdir(exist_ok=True)
    rng = np.random.default_rng(77)
    pts = dataio.PointSampleSet(locations=rng.uniform(-0.95, 0.95, (50, 3)),
                                values=rng.normal(size=(50, 2)))
    dataio.save_points(str(OUT / "points.fcpt"), pts)
    dataio.save_points(str(OUT / "points.csv"), pts)
    ck = dataio.Checkpoint(levels=5, rho=4, kernel="gaussian", alpha=1000.0,
                           p=rng.uniform(-0.9, 0.9, (40, 3)), w=rng.normal(size=(40, 4)),
                           bias=0.0625)
    dataio.save_checkpoint(str(OUT / "sdf.ckpt"), ck)
    cams = [(Camera(position=np.array([0.3, -0.2, -2.5]), look_at=np.array([0.0, 0.1, 0.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_deg=40.0, width=16, height=12), "f0.ppm"),
            (Camera(position=np.array([2.0, 0.5, 0.0]), look_at=np.zeros(3),
                    up=np.array([0.0, 0.0, 2.0]), fov_deg=55.5, width=8, height=8), None)]
    dataio.save_cameras(str(OUT / "cams.json"), cams)
    img = rng.uniform(-0.1, 1.1, (5, 7, 3))
    img[0, 0] = [0.5, 1.0 / 510.0, 0.0]
    dataio.save_image(str(OUT / "img.ppm"), img)
    back_pts = dataio.load_points(str(OUT / "points.fcpt"))
    back_cams = dataio.load_cameras(str(OUT / "cams.json"))
    np.savez_compressed(
        OUT.parent / "io.npz", locations=back_pts.locations, values=back_pts.values,
        ckpt_p=ck.p, ckpt_w=ck.w, ckpt_bias=np.array(ck.bias), img_src=img,
        img_back=dataio.load_image(str(OUT / "img.ppm")),
        cam_pos=np.stack([c.position for c, _ in back_cams]),
        cam_look=np.stack([c.look_at for c, _ in back_cams]),
        cam_up=np.stack([c.up for c, _ in back_cams]))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
