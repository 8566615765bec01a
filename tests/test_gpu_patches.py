"""GPU parity: N-D extraction, coverage and overlap-add vs the oracle and the
reference-generated fixtures (tests/golden/extract_cases.npz).

Bars: patch order, observed flags, origins, coverage and uncovered handling are
BIT-EXACT; values/means/reconstructions (f32 on device vs f64 reference) within
abs 1e-6 (values in [0,1]-scaled units) — stated tolerance.
"""

import numpy as np
import pytest
import torch

from oracle import patches as op
from paper_2311_15061_b200 import patches as pp

pytestmark = pytest.mark.gpu
TOL = 1e-6


def test_golden_cases(golden, cuda_device):
    g = golden("extract_cases.npz")
    for ci in range(int(g["num_cases"])):
        p = f"c{ci}_"
        spec = pp.PatchSpec(tuple(g[p + "patch"]), tuple(g[p + "stride"]))
        pm = pp.extract_patches(g[p + "tensor"], g[p + "mask"], spec, bool(g[p + "mean_subtract"]))
        vals, obs, means = pm.to_host()
        assert np.array_equal(obs, g[p + "observed"]), ci
        assert np.array_equal(pm.origins, g[p + "origins"]), ci
        assert np.abs(vals - g[p + "values"]).max(initial=0) <= TOL, ci
        assert np.abs(means - g[p + "means"]).max(initial=0) <= TOL, ci
        assert np.array_equal(vals[~obs], np.zeros((~obs).sum())), "unobserved must be exactly 0"
        assert np.array_equal(pp.coverage_map(pm), g[p + "coverage"]), ci
        assert pm.n_obs == int(g[p + "observed"].sum())
        rec = pp.reconstitute(pm, g[p + "est"])
        assert rec.dtype == np.float64 and rec.shape == g[p + "recon"].shape
        assert np.abs(rec - g[p + "recon"]).max() <= 1e-5, ci


def test_extract_2x2_stride_2_exact(cuda_device):
    t = np.arange(16, dtype=float).reshape(4, 4)
    pm = pp.extract_patches(t, np.ones((4, 4), bool), pp.PatchSpec((2, 2), (2, 2)))
    v, _, m = pm.to_host()
    assert v[0].tolist() == [0, 1, 4, 5] and v[3].tolist() == [10, 11, 14, 15]
    assert np.all(m == 0)


def test_mean_subtraction_uses_observed_only(cuda_device):
    t = np.array([[1.0, 3.0], [100.0, 5.0]])
    mask = np.array([[True, True], [False, True]])
    pm = pp.extract_patches(t, mask, pp.PatchSpec((2, 2)), mean_subtract=True)
    v, _, m = pm.to_host()
    assert m[0] == pytest.approx(3.0)
    assert v[0].tolist() == [-2.0, 0.0, 0.0, 2.0]


def test_unobserved_values_never_leak(cuda_device):
    rng = np.random.default_rng(1)
    t = rng.random((6, 6))
    mask = rng.random((6, 6)) < 0.5
    garbage = t.copy()
    garbage[~mask] = rng.random((~mask).sum()) * 1e6
    for ms in (False, True):
        a = pp.extract_patches(t, mask, pp.PatchSpec((3, 3)), ms)
        b = pp.extract_patches(garbage, mask, pp.PatchSpec((3, 3)), ms)
        assert torch.equal(a.values_pn, b.values_pn) and torch.equal(a.means_dev, b.means_dev)


@pytest.mark.parametrize("shape,patch,stride", [((7, 9), (3, 3), (1, 1)), ((8, 8), (4, 2), (2, 2)),
                                                ((5, 5, 3), (2, 2, 3), (1, 1, 1)), ((16,), (4,), (2,)),
                                                ((5, 4, 3, 4), (2, 2, 3, 2), (1, 2, 1, 1))])
def test_roundtrip_identity_bitwise_on_integers(cuda_device, shape, patch, stride):
    rng = np.random.default_rng(2)
    t = rng.integers(0, 256, size=shape).astype(np.float64)
    pm = pp.extract_patches(t, np.ones(shape, bool), pp.PatchSpec(patch, stride))
    rec = pp.reconstitute(pm, pm.values)
    cov = pp.coverage_map(pm) > 0
    assert np.array_equal(rec[cov], t[cov])


def test_reconstitute_matches_oracle_random(cuda_device):
    rng = np.random.default_rng(5)
    for shape, patch, stride, ms in [((37, 41), (8, 8), (1, 1), True), ((12, 10, 6), (4, 3, 6), (2, 1, 1), False),
                                     ((64, 64), (10, 10), (3, 2), True)]:
        t = rng.random(shape)
        mask = rng.random(shape) < 0.3
        pm = pp.extract_patches(t, mask, pp.PatchSpec(patch, stride), ms)
        opm = op.extract_patches(t, mask, patch, stride, ms)
        est = rng.standard_normal(opm.values.shape)
        got = pp.reconstitute(pm, est)
        want = op.reconstitute(opm, est)
        assert np.abs(got - want).max() <= 1e-5
        # fused data consistency
        got_dc = pp.reconstitute(pm, est, dc_original=t, dc_mask=mask)
        assert np.array_equal(got_dc[mask], t[mask])
        assert np.abs(got_dc[~mask] - want[~mask]).max() <= 1e-5


def test_strict_coverage_error(cuda_device):
    pm = pp.extract_patches(np.zeros((5, 5)), np.ones((5, 5), bool), pp.PatchSpec((2, 2), (2, 2)))
    with pytest.raises(pp.CoverageError):
        pp.reconstitute(pm, pm.values, strict=True)
    out = pp.reconstitute(pm, pm.values)
    assert np.all(out[4, :] == 0) and np.all(out[:, 4] == 0)


def test_shape_errors(cuda_device):
    t = np.zeros((4, 4))
    with pytest.raises(pp.ShapeError):
        pp.extract_patches(t, np.ones((3, 4), bool), pp.PatchSpec((2, 2)))
    with pytest.raises(pp.ShapeError):
        pp.extract_patches(t, np.ones((4, 4), bool), pp.PatchSpec((5, 2)))
    pm = pp.extract_patches(t, np.ones((4, 4), bool), pp.PatchSpec((2, 2)))
    with pytest.raises(pp.ShapeError):
        pp.reconstitute(pm, np.zeros((3, 4)))


def test_large_frame_indices_exact(cuda_device):
    """cfg-3-sized frame (512^2, 8x8, line-hop): observed flags and coverage exact."""
    from paper_2311_15061_b200 import inputs

    img = inputs.synthetic_texture((512, 512), seed=0)
    mask = inputs.make_mask((512, 512), 0.25, "line-hop", 0)
    pm = pp.extract_patches(img, mask, pp.PatchSpec((8, 8)), True)
    opm = op.extract_patches(img, mask, (8, 8), (), True)
    _, obs, means = pm.to_host()
    assert np.array_equal(obs, opm.observed)
    assert np.abs(means - opm.means).max() <= TOL
    assert np.array_equal(pp.coverage_map(pm), op.coverage((512, 512), (8, 8), (1, 1)))


def _w_row_off(il):
    """Byte offset of row il's first chunk in a W tile block (pb_index.cuh w_row_off)."""
    il = np.asarray(il, dtype=np.int64)
    return ((il >> 2) << 7) | ((((il & 3) << 1) ^ ((il >> 2) & 7)) << 4)


def _w_row_index(off):
    """Inverse of _w_row_off."""
    line = off >> 7
    return line * 4 + ((((off >> 4) & 7) ^ (line & 7)) >> 1)


def test_w_row_offset_is_a_bijection():
    il = np.arange(1024)
    off = _w_row_off(il)
    assert len(np.unique(off)) == 1024 and off.max() < 2 ** 15 and np.all(off % 16 == 0)
    assert np.array_equal(_w_row_index(off), il)


def _carve(buf, n, p, nnz):
    """Mirror of carve_index (pb_index.cu) to read the index back for checking."""
    kt = 1024
    nt = -(-n // kt)
    ecap = 2 * nnz + 6144 * nt + 1024                              # ell_cap
    wcap = nt * (8 + (2 * p + 31) // 32) + 2 * nnz // 1024 + 1     # wave_cap
    out, off = {}, 0
    for name, cnt, dt in [("tile_tot", nt, np.int32), ("tile_base", nt + 1, np.int64),
                          ("colptr", nt * ((p + 1 + 3) & ~3), np.int32), ("rowptr", n + 1, np.int64),
                          ("e_loc", nnz, np.uint16), ("x_csc", ecap, np.float32), ("csr_p", nnz, np.uint16),
                          ("csr_pos", nnz, np.uint32), ("cmax", 16, np.int32), ("outliers", n, np.int32),
                          ("out_tot", nt, np.int32), ("out_base", nt + 1, np.int64), ("hist", p + 2, np.int32),
                          ("tile_segs", nt, np.int32), ("seg_base", nt + 1, np.int64),
                          ("slot_csc", nnz, np.uint32), ("e_ell", ecap, np.uint16), ("ell_tot", nt, np.int32),
                          ("ell_base", nt + 1, np.int64), ("wave_tot", nt, np.int32), ("wave_base", nt + 1, np.int64),
                          ("wave_off", wcap, np.uint32), ("wave_meta", wcap, np.uint16),
                          ("wave_col", wcap * 32, np.uint16)]:
        nb = cnt * np.dtype(dt).itemsize
        out[name] = buf[off:off + nb].view(dt)
        off += (nb + 255) & ~255
    return out


@pytest.mark.parametrize("shape,patch,ratio,kind", [((40, 45), (8, 8), 0.25, "uniform-random"),
                                                     ((70, 64), (8, 8), 0.25, "line-hop"),
                                                     ((50, 41), (10, 10), 0.1, "uniform-random"),
                                                     ((12, 10, 6), (4, 3, 6), 0.3, "uniform-random"),
                                                     ((300, 40), (10, 10), 0.1, "uniform-random")])
def test_observed_element_index_exact(cuda_device, shape, patch, ratio, kind):
    """The observed-element index (pb_index.cu) element by element: the CSR
    view (ascending offsets per patch), and the dictionary step's ELL wave
    layout — every observed element at exactly one position of its tile's
    range, in a lane whose run belongs to its column, each column in one wave
    per tile on R aligned lanes (uniform R per wave), padding pointing at the
    zero W row with value 0, and bank-spread quarter-warp steps."""
    from paper_2311_15061_b200 import inputs

    rng = np.random.default_rng(0)
    img = rng.random(shape)
    mask = inputs.make_mask(shape, ratio, kind, 3)
    pm = pp.extract_patches(img, mask, pp.PatchSpec(patch), True)
    ix = pm.index()
    vals, obs, _ = pm.to_host()
    n, p = obs.shape
    assert ix.nnz == obs.sum() and ix.cmax == obs.sum(1).max()
    b = _carve(pm._cache["ix_buf"].cpu().numpy(), n, p, int(ix.nnz))
    rows, cols = np.nonzero(obs)          # row-major => ascending (i, p)
    assert np.array_equal(b["csr_p"].astype(np.int64), cols)
    assert np.array_equal(b["rowptr"][:n], np.concatenate([[0], np.cumsum(obs.sum(1))[:-1]]))
    pos = b["csr_pos"].astype(np.int64)
    nell = int(b["ell_base"][-1])
    assert nell == ix.nnz_ell and len(np.unique(pos)) == len(pos) and pos.max(initial=0) < nell
    tile = rows // 1024
    assert np.array_equal(b["e_ell"][pos].astype(np.int64), _w_row_off(rows - tile * 1024))
    assert np.array_equal(b["x_csc"][pos], vals[rows, cols].astype(np.float32))
    eb, wb = b["ell_base"].astype(np.int64), b["wave_base"].astype(np.int64)
    assert np.all((pos >= eb[tile]) & (pos < eb[tile + 1]))
    pad = np.ones(nell, bool)
    pad[pos] = False
    assert np.all(b["e_ell"][:nell][pad] == 32768) and np.all(b["x_csc"][:nell][pad] == 0)
    # wave of each element and its lane's column
    woff, meta, wcol = b["wave_off"].astype(np.int64), b["wave_meta"].astype(np.int64), b["wave_col"].astype(np.int64)
    rel = pos - eb[tile]
    for t in np.unique(tile):
        ws = np.arange(wb[t], wb[t + 1])
        sel = tile == t
        w = ws[np.searchsorted(woff[ws], rel[sel], side="right") - 1]
        lane = (rel[sel] - woff[w]) % 32
        step = (rel[sel] - woff[w]) // 32
        assert np.all(step < (meta[w] & 0xFF))
        assert np.array_equal(wcol[w * 32 + lane], cols[sel])
        cols_seen = []
        for wv in ws:
            c = wcol[wv * 32:(wv + 1) * 32]
            r = 1 << (meta[wv] >> 8)
            for g in range(0, 32, r):
                grp = c[g:g + r]
                assert np.all(grp == grp[0]), (wv, g, grp)
                if grp[0] != 0xFFFF:
                    cols_seen.append(int(grp[0]))
        assert len(cols_seen) == len(set(cols_seen))      # one wave per column per tile
    # bank spreading: W-row bank quads inside each quarter-warp step (1 = conflict
    # free) against the same runs filled in ascending patch order
    def quarter_cost(blk):
        cost = 0
        for qtr in range(4):
            e = blk[:, 8 * qtr: 8 * qtr + 8]
            for jj in range(e.shape[0]):
                q = (e[jj][e[jj] != 32768] >> 4) & 7
                cost += np.bincount(q, minlength=8).max() if len(q) else 0
        return cost

    spread = ascending = 0
    for t in range(len(wb) - 1):
        for wv in range(wb[t], wb[t + 1]):
            lw = int(meta[wv] & 0xFF)
            blk = b["e_ell"][eb[t] + woff[wv]: eb[t] + woff[wv] + 32 * lw].astype(np.int64).reshape(lw, 32)
            asc = np.full_like(blk, 32768)
            r = 1 << (meta[wv] >> 8)
            for g in range(0, 32, r):
                el = blk[:, g:g + r].ravel()
                el = _w_row_off(np.sort(_w_row_index(el[el != 32768])))
                for k, e in enumerate(el):
                    asc[k // r, g + k % r] = e
            spread += quarter_cost(blk)
            ascending += quarter_cost(asc)
    assert spread <= ascending, (spread, ascending)


@pytest.mark.parametrize("shape,patch,stride,f32", [((70, 1100), (10, 10), (1, 1), False),   # wide: row tiles
                                                    ((300, 800), (8, 8), (1, 1), True),
                                                    ((45, 333), (6, 5), (1, 1), False),     # runtime shape
                                                    ((64, 64), (10, 10), (3, 1), False),    # row stride > 1
                                                    ((64, 90), (7, 7), (2, 3), True),       # fallback OLA
                                                    ((9, 300), (10, 10), (1, 1), False)])   # < one patch row of
def test_rank2_fast_paths_bit_identical_to_generic(cuda_device, shape, patch, stride, f32):   # output rows
    """The rank-2 kernels (shared-memory windows for extraction, staged runs for
    overlap-add) against the generic N-D kernels on the same frame viewed as
    (1, H, W): identical values, flags, means and reconstructions, bit for bit
    (same per-element arithmetic and the same ascending patch order)."""
    rng = np.random.default_rng(11)
    if shape[0] < patch[0]:
        patch = (shape[0], patch[1])
    t = rng.random(shape)
    mask = rng.random(shape) < 0.2
    dt = torch.float32 if f32 else torch.float64
    tt = torch.as_tensor(t, dtype=dt, device="cuda")
    mm = torch.as_tensor(mask, device="cuda")
    pm2 = pp.extract_patches(tt, mm, pp.PatchSpec(patch, stride), True)
    pm3 = pp.extract_patches(tt[None], mm[None], pp.PatchSpec((1,) + patch, (1,) + stride), True)
    assert torch.equal(pm2.values_pn, pm3.values_pn)
    assert torch.equal(pm2.observed_pn, pm3.observed_pn)
    assert torch.equal(pm2.means_dev, pm3.means_dev) and torch.equal(pm2.counts, pm3.counts)
    est = torch.randn(pm2.values_pn.shape, device="cuda")
    for dc in (False, True):
        kw = dict(dc_original=tt, dc_mask=mm) if dc else {}
        kw3 = dict(dc_original=tt[None], dc_mask=mm[None]) if dc else {}
        r2 = pp.reconstitute(pm2, est.T, out="device", dtype=dt, **kw)
        r3 = pp.reconstitute(pm3, est.T, out="device", dtype=dt, **kw3)
        assert torch.equal(r2, r3[0]), (shape, patch, stride, dc)
