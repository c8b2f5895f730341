"""Loader for tests/golden/golden_v1.npz (written by tests/golden/make_golden.py)."""

import functools
import json
import os

import numpy as np

from oracle.adpsplit_oracle import Cam, Gaussians

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_v1.npz")


@functools.lru_cache(maxsize=1)
def load():
    z = np.load(PATH)
    data = {k: z[k] for k in z.files}
    meta = json.loads(str(data.pop("meta_json")))
    return data, meta


def scene(data, prefix):
    return (Gaussians(data[f"{prefix}__mu"], data[f"{prefix}__scale"], data[f"{prefix}__rot"],
                      data[f"{prefix}__opacity"], data[f"{prefix}__sh_dc"],
                      data[f"{prefix}__sh_rest"]),
            float(data[f"{prefix}__extent"]))


def cams(data, key):
    return [Cam.from_row(r) for r in data[key]]


class Cfg:
    def __init__(self, d):
        self.__dict__.update(d)
