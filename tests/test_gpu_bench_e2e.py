"""bench.py's end-to-end pipeline (host inputs, chunked uploads / GEMMs / read-backs, per-tensor
sync) must produce exactly the device-resident step's outputs: same quantizers, same GEMM per
row (row blocks of a GEMM are independent), so the read-back BF16 outputs are bitwise equal."""
import pytest
import torch

pytestmark = pytest.mark.gpu


# row blocks of > 256 rows: the device step and every block run the same (CTA-pair) GEMM kernel,
# whose per-element arithmetic does not depend on M (blocks of <= 256 rows can take the decode
# kernel, whose cluster split-K sums k-ranges in another order: equal only to ~1 ulp)
@pytest.mark.parametrize("m,chunks", [(2048, 4), (1536, 3)])
def test_e2e_pipeline_equals_device_step(m, chunks):
    import bench
    dev = torch.device("cuda", 0)
    st = bench.LayerStep(1, 0, dev, m=m)
    st.run()
    torch.cuda.synchronize()
    ref = {k: v.clone() for k, v in st.y.items()}
    for v in st.y.values():
        v.zero_()
    st.run_e2e(chunks=chunks)
    torch.cuda.synchronize()
    st.engine.check_finite()
    for name, y in ref.items():
        got, want = st.h_y[name], y.cpu()
        bad = (got.view(torch.int16) != want.view(torch.int16))
        if bad.any():
            rows = bad.any(dim=1).nonzero().flatten()
            d = (got.float() - want.float()).abs().max().item()
            raise AssertionError(f"{name}: {int(bad.sum())} differ, rows {rows[:8].tolist()}..{rows[-3:].tolist()} "
                                 f"({rows.numel()} rows), max |diff| {d}")
