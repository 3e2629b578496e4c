"""GPU: contact penalty + friction terms of the colour pass (_native.pyx:351-399, DCD anchors
refreshed :134-172) through vbd_set_contacts, against passes recorded at the reference's own
kernel seam (tests/golden/contact_scene.npz).  Bars: fp64 1e-12 absolute (the reference's
native-vs-NumPy bar), fp32 1e-5 absolute (scene span 0.5, contact stiffness 1e6)."""

import numpy as np
import pytest

from extras import ContactCall, contact_system

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def V():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2403_06321_b200 as V
    return V


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
def test_contact_passes_match_reference(V, O, golden, precision, tol):
    g = golden("contact_scene.npz")
    s = contact_system(O)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision=precision)
    h = float(g["h"])
    for k in range(int(g["num_calls"])):
        c = ContactCall(g, k)
        ctx.set_contacts(c, float(g[f"call{k}_mu_c"]), float(g[f"call{k}_eps_v"]))
        x = g[f"call{k}_x0"].copy()
        ctx.color_pass(x, g[f"call{k}_x_t"], g[f"call{k}_y"], h, g[f"call{k}_group"])
        err = np.abs(x - g[f"call{k}_x1"]).max()
        assert err <= tol, (k, err)
    # with the contact set cleared, the passes where contacts are active (gap d > 0) differ
    ctx.set_contacts(None)
    diffs = []
    for k in range(int(g["num_calls"])):
        x = g[f"call{k}_x0"].copy()
        ctx.color_pass(x, g[f"call{k}_x_t"], g[f"call{k}_y"], h, g[f"call{k}_group"])
        diffs.append(np.abs(x - g[f"call{k}_x1"]).max())
    assert max(diffs) > 5 * tol, diffs


def test_contact_line_search_vs_oracle(V, O, golden):
    g = golden("contact_scene.npz")
    s = contact_system(O)
    ctx = V.DeviceContext.from_system(O.RefSystemView(s), precision="fp64")
    h = float(g["h"])
    for k in (0, 6):
        c = ContactCall(g, k)
        mu, ev = float(g[f"call{k}_mu_c"]), float(g[f"call{k}_eps_v"])
        ctx.set_contacts(c, mu, ev)
        a = g[f"call{k}_x0"].copy()
        b = a.copy()
        ctx.color_pass(a, g[f"call{k}_x_t"], g[f"call{k}_y"], h, g[f"call{k}_group"], line_search=True)
        O.color_pass(s, b, g[f"call{k}_x_t"], g[f"call{k}_y"], h, g[f"call{k}_group"],
                     line_search=True, carr=c, mu_c=mu, eps_v=ev)
        assert np.abs(a - b).max() <= 1e-12, k
