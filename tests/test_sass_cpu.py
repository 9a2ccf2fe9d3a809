"""The built library is sm_100a code on the intended hardware units (no GPU needed: cuobjdump
reads the SASS of libkx.so).  B200_PROFILING.md: SASS mnemonics are the proof — DMMA for the
fp64 tensor-core mode products, LDGSTS for the cp.async pipeline, SYNCS for the mbarrier
pipeline, UCGABAR for the thread-block-cluster barriers of the small-grid and cluster split-K
kernels; no legacy half-precision HMMA anywhere (the path is fp64)."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2310_07551_b200", "libkx.so")


@pytest.fixture(scope="module")
def sass():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    if not os.path.exists(LIB):
        from paper_2310_07551_b200 import build
        build.build()
    r = subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-500:]
    return r.stdout


def _functions(sass, pattern):
    """SASS text of every function whose mangled name matches pattern."""
    out, cur, keep = [], [], False
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            if keep:
                out.append("\n".join(cur))
            cur, keep = [line], re.search(pattern, m.group(1)) is not None
        elif keep:
            cur.append(line)
    if keep:
        out.append("\n".join(cur))
    return out


def test_sm100a_only(sass):
    arches = set(re.findall(r"arch = (sm_\w+)", sass))
    assert arches == {"sm_100a"}, arches


def test_mode_product_gemm_uses_fp64_tensor_cores(sass):
    gemms = _functions(sass, r"11gemm_kernelI")   # the fp64 template (not the tf32 kernel)
    assert len(gemms) >= 12          # 3 tile configs x 2 layouts x 2 vector widths (+ peer stores)
    tma = _functions(sass, r"11gemm_kernelILi128ELi128ELi32ELi32ELi32ELb[01]ELi3E")   # VEC = 3
    assert len(tma) == 2             # the opt-in TMA-fed 128x128x32 variant, both layouts
    for f in gemms:
        assert "DMMA.8x8x4" in f      # fp64 tensor-core MMA
        assert "SYNCS" in f           # mbarrier full/empty pipeline
        assert "HMMA" not in f
        if f in tma:
            assert "UTMALDG" in f and "LDGSTS" not in f   # tensor-map loads, no cp.async
        else:
            assert "LDGSTS" in f      # cp.async shared-memory pipeline
    # the cluster split-K path: thread-block cluster barriers in the GEMM
    assert any("UCGABAR" in f for f in gemms)


def test_small_grid_kernels_use_clusters_and_dmma(sass):
    fused = _functions(sass, "fused2d_kernel")
    assert len(fused) == 1
    assert "DMMA.8x8x4" in fused[0] and "UCGABAR_ARV" in fused[0] and "UCGABAR_WAIT" in fused[0]
    tucker = _functions(sass, "tucker2d_small_kernel")
    assert len(tucker) == 1 and "DMMA.8x8x4" in tucker[0]


def test_no_half_precision_mma_in_fp64_path(sass):
    """Only the fp32 variant's kernel (tf32x3_gemm_kernel) may use the tcgen05 tensor cores."""
    rest = _functions(sass, r"^(?!.*tf32x3_gemm_kernel)")
    assert rest
    for f in rest:
        assert "HMMA" not in f and not re.search(r"UTC\w*MMA", f)


def test_fp32_gemm_is_tcgen05_with_tma(sass):
    """fp32 variant: tcgen05 MMA (UTC*MMA) fed by TMA tensor loads (UTMALDG),
    accumulators read back from TMEM (LDTM), TMEM allocated/freed by the kernel."""
    fs = _functions(sass, r"tf32x3_gemm_kernel")
    assert len(fs) == 2              # persistent and cluster split-K instantiations
    for f in fs:
        assert re.search(r"UTC\w*MMA", f)
        assert "UTMALDG" in f
        assert "LDTM" in f
        assert "DMMA" not in f
    assert any("UCGABAR" in f for f in fs)   # the split variant's cluster barriers
    assert any("UTMASTG" in f for f in fs)   # the persistent variant's TMA output stores


def test_peer_store_gemms_fence_at_system_scope(sass):
    """The GEMM instantiations that store straight into other ranks' buffers (the fused
    all-to-all) end with a system-scope fence; the plain ones do not pay for it."""
    peer = _functions(sass, r"gemm_kernel.*Li3ELb1E")     # ..., STAGES = 3, PEER = true
    plain = _functions(sass, r"gemm_kernel.*Li3ELb0E")
    assert len(peer) >= 6 and len(plain) >= 6
    assert all("MEMBAR.SC.SYS" in f for f in peer)
    assert not any("MEMBAR.SC.SYS" in f for f in plain)
