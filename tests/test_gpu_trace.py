"""hmat_cta_trace: per-CTA [start, end, SM] records of the last launches."""
import numpy as np
import pytest

from gen import hgen
from gen.hgen import HConfig
from tests.helpers import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2008_12441_b200 import hmat as hm


@pytest.mark.parametrize("nrhs", [1, 64])
def test_cta_trace_records(nrhs):
    cfg = HConfig("tr", d=3, L=3, b=64, r=32, nrhs=nrhs, seed=601)
    U, V, D = hgen.inputs(cfg)
    h = hm.hmat_create(cfg.L, cfg.d, cfg.b, cfg.r, U, V, D)
    try:
        x = torch.from_numpy(np.ascontiguousarray(hgen.xblock(cfg, nrhs=nrhs).T)).cuda()
        y0, y1 = torch.empty_like(x), torch.empty_like(x)
        hm.hmat_matvec(h, x.t(), y0.t(), nrhs)
        with pytest.raises(hm.HMatError):
            hm.hmat_cta_trace_read(h, 0)           # not enabled
        hm.hmat_cta_trace(h, True)
        hm.hmat_matvec(h, x.t(), y1.t(), nrhs)
        nsm = torch.cuda.get_device_properties(0).multi_processor_count
        for k in (0, 1):
            recs = hm.hmat_cta_trace_read(h, k)
            assert len(recs) > 0
            ran = [r for r in recs if r[1] > 0]
            assert len(ran) >= 1
            assert all(r[1] >= r[0] > 0 and 0 <= r[2] < nsm for r in ran)
        hm.hmat_cta_trace(h, False)
        assert torch.equal(y0, y1)                 # tracing does not change the result
        assert_parity(y1.t().cpu().numpy(), y0.t().cpu().numpy())
    finally:
        hm.hmat_destroy(h)
