"""PSNR / max-abs of forward_full against the reference golden (tests/golden/net_small.npz)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import fovray_oracle as O  # noqa: E402
from paper_2209_09965_b200 import network as N  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "net_small.npz")
for tag, blocks, seed, frames in (("full", N.FULL_BLOCKS, 0, 3), ("fullwide", N.FULL_BLOCKS, 3, 2)):
    net = N.quantized_net(N.init_network(N.NetConfig.from_string(blocks), seed=seed), "fp16")
    state = N.reset_state(net.config, g[f"{tag}_x0"].shape[2:])
    for f in range(frames):
        o, od, state = N.forward_full(net, g[f"{tag}_x{f}"], state)
        ref = g[f"{tag}_o{f}"]
        q = O.psnr(np.moveaxis(o.data[0], 0, -1), np.moveaxis(ref[0], 0, -1))
        print(f"{tag} frame {f}: PSNR {q:.2f} dB, max |o - ref| {np.abs(o.data - ref).max():.2e}")
