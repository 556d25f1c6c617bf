"""bench.py's end-to-end pipeline (host inputs, chunked uploads / GEMMs / read-backs, per-tensor
sync) must produce the device-resident step's outputs: same quantizers, same GEMM per row (row
blocks of a GEMM are independent), so the read-back BF16 outputs are bitwise equal -- except
where one of the two GEMM calls cuts its tail-wave tiles into K slices (gemm.cu plan_split: it
depends on the tile count, i.e. on M), which changes the fp32 summation order: there the BF16
outputs agree to one BF16 ulp (plus fp32
reordering error on cancelling sums)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


# the bench configuration itself (M = 8192 in 4 blocks of 2,048 rows): the device step and every
# block run the CTA-pair kernel, whose per-element arithmetic does not depend on M (other block
# sizes can select the decode kernel or a split-K plan, which sum k-ranges in another order)
@pytest.mark.parametrize("m,chunks", [(8192, 4)])
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
    from paper_2601_18150_b200 import fp8q
    lib = fp8q.load_library()
    for name, y in ref.items():
        got, want = st.h_y[name], y.cpu()
        n, kk = y.shape[1], st.xq[name].shape[1]
        if lib.fp8_block_gemm_workspace_size(m, n, kk) != lib.fp8_block_gemm_workspace_size(m // chunks, n, kk):
            gf, wf = got.float(), want.float()
            ulp = torch.ldexp(torch.ones_like(wf), torch.frexp(wf.abs().clamp_min(1e-30))[1] - 8)
            # one BF16 ulp, plus fp32 reordering error for cancelling sums (relative to the row)
            tol = ulp + 1e-5 * wf.abs().amax(dim=1, keepdim=True)
            assert ((gf - wf).abs() <= tol).all(), (name, float(((gf - wf).abs() - tol).max()))
            assert (gf != wf).float().mean().item() < 0.01, name
            continue
        bad = (got.view(torch.int16) != want.view(torch.int16))
        if bad.any():
            rows = bad.any(dim=1).nonzero().flatten()
            d = (got.float() - want.float()).abs().max().item()
            raise AssertionError(f"{name}: {int(bad.sum())} differ, rows {rows[:8].tolist()}..{rows[-3:].tolist()} "
                                 f"({rows.numel()} rows), max |diff| {d}")
