"""se1p_set_allocator (include/se1p.h; SURVEY.md 8(b) "Ownership"): the library's plans,
workspaces and tables come from torch's caching allocator when the hook is installed, results
are bitwise those of the cudaMalloc path, and switching back returns the memory."""
import pytest

from se1p_synth import make_system

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1611_09538_b200 as se1p  # noqa: E402


def test_torch_allocator_hook():
    L = (1.0, 1.0, 1.0)
    x, q = make_system(2000, L, 31)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    kw = dict(n_local=3, S0=416, SI=416, Ntilde=64)
    se1p.use_torch_allocator(False)
    a = se1p.kspace(xd, qd, L, 8.0, 32, 20, **kw)
    ra = se1p.real(xd, qd, L, 8.0, 0.594)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    try:
        se1p.use_torch_allocator(True)
        b = se1p.kspace(xd, qd, L, 8.0, 32, 20, **kw)
        rb = se1p.real(xd, qd, L, 8.0, 0.594)
        g = se1p.kspace(xd, qd, L, 8.0, 32, 20, graph=True, **kw)   # graphs bake the hook's pointers
        g = se1p.kspace(xd, qd, L, 8.0, 32, 20, graph=True, **kw)
        torch.cuda.synchronize()
        held = torch.cuda.memory_allocated() - base
        # the workspace (real grid, planes, kernel spectra, records) now lives in torch's pool
        info = se1p.plan_info(L, 8.0, 32, 20, **kw)
        assert held >= info["grid_points"] * 8, held
    finally:
        se1p.use_torch_allocator(False)
    torch.cuda.synchronize()
    outputs = sum(((t.numel() * 8 + 511) // 512) * 512 for t in (b, rb, g))
    assert torch.cuda.memory_allocated() - base <= outputs   # the library's memory went back
    assert torch.equal(a, b) and torch.equal(a, g) and torch.equal(ra, rb)
    # and the default path still works afterwards
    assert torch.equal(se1p.kspace(xd, qd, L, 8.0, 32, 20, **kw), a)
