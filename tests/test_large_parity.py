"""Large-scale parity pins on CPU: the product's generators rebuild exactly
the instances the reference planned for tests/golden/huge.json, and the C
oracle reproduces the reference's own plans there (so the GPU tests that
compare against the oracle at these sizes compare against the reference)."""
import numpy as np
import pytest

import oracle
from conftest import family_instance, lstm_instances, sha64


@pytest.mark.parametrize("name", ["uniform_1e5_s0", "cnn_1e5_s0", "walk_1e5_s0",
                                  "uniform_1e5_s1", "walk_1e5_s1"])
def test_generators_rebuild_reference_instances(huge_golden, name):
    a, f, s = family_instance(name)
    g = huge_golden[name]
    assert len(a) == g["n"]
    assert sha64(np.stack([s, a, f], 1)) == g["blocks_sha256"]


@pytest.mark.parametrize("layers,align", [(6, 512), (64, 512), (6, 1), (64, 1)])
def test_lstm_oracle_matches_reference_digest(huge_golden, layers, align):
    tp, a, f, s = lstm_instances(layers, align)
    g = huge_golden[f"lstm_L{layers}" + ("_a512" if align == 512 else "")]
    assert sha64(np.stack([s, a, f], 1)) == g["blocks_sha256"]
    offs, peaks = [], []
    for t in range(len(tp) - 1):
        o, p = oracle.solve_bestfit(a[tp[t]:tp[t + 1]], f[tp[t]:tp[t + 1]], s[tp[t]:tp[t + 1]])
        offs.append(o)
        peaks.append(p)
    assert sha64(np.concatenate(offs)) == g["offsets_sha256"]
    assert sha64(np.asarray(peaks)) == g["peaks_sha256"]


@pytest.mark.parametrize("name", ["walk_1e5_s0", "cnn_1e5_s0"])
def test_oracle_matches_reference_at_1e5(huge_golden, name):
    a, f, s = family_instance(name)
    off, peak = oracle.solve_bestfit(a, f, s)
    g = huge_golden[name]
    assert peak == g["peak"] and sha64(off) == g["offsets_sha256"]
