"""Dataset files written by the UNMODIFIED reference (splatsched-v1,
/root/reference/pkg/src/splatsched/scene.py:468-528).

Run in the build container only (needs /root/reference):
    python tests/golden/make_dataset_golden.py
Writes tests/golden/dataset_v1/{aerial,temporal,street}/ (dataset.json +
points.bin); tests/test_dataset.py checks that paper_2512_20017_b200.dataset
writes the same bytes and reads them back.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def main():
    tmp = tempfile.mkdtemp(prefix="refpkg_")
    shutil.copytree(os.path.join(REF, "splatsched"), os.path.join(tmp, "splatsched"))
    sys.path.insert(0, tmp)
    import splatsched as ss

    out = os.path.join(HERE, "dataset_v1")
    shutil.rmtree(out, ignore_errors=True)
    cases = {
        "aerial": ss.generate_aerial_scene(seed=3, n_points=60, grid=(2, 2), n_views=3, altitude=25),
        "temporal": ss.generate_aerial_scene(seed=4, n_points=40, grid=(1, 2), n_views=4, altitude=20, duration=5.0),
        "street": ss.generate_street_scene(seed=11, n_points=50, trajectory_waypoints=[(0, 0, 2), (40, 0, 2), (40, 30, 2)],
                                           n_views=4),
    }
    for name, ds in cases.items():
        ss.save_dataset(ds, os.path.join(out, name))
    print("wrote", out)


if __name__ == "__main__":
    main()
