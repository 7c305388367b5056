import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

ASSETS = os.path.join(ROOT, "assets", "generated")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


def ensure_assets():
    """Models/clips are generated deterministically (tools/gen_assets.py)."""
    need = ["arm2_m6.json", "arm2_m6_sine.csv", "pendulum1_m2.json", "walker5_m16.json", "wb700.json",
            "wb700_fixed.json", "wb700_dance.csv", "wb700_backflip.csv", "wb700_fixed_dance.csv",
            "wb700_general.json", "wb700_slow.json"]
    if not all(os.path.exists(os.path.join(ASSETS, n)) for n in need):
        from tools.gen_assets import generate
        generate(ASSETS)
    return ASSETS


@pytest.fixture(scope="session")
def assets():
    return ensure_assets()


def model_paths(name):
    clip = {"pendulum1_m2": "pendulum1_m2_sine", "arm2_m6": "arm2_m6_sine", "walker5_m16": "walker5_m16_sine",
            "wb700": "wb700_dance", "wb700_fixed": "wb700_fixed_dance", "wb700_backflip": "wb700_backflip",
            "wb700_general": "wb700_fixed_dance", "wb700_slow": "wb700_dance"}[name]
    model = "wb700" if name == "wb700_backflip" else name
    return os.path.join(ASSETS, model + ".json"), os.path.join(ASSETS, clip + ".csv")
