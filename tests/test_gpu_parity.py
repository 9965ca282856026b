"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Index work (stage outputs, masks) must be bit-exact; attention outputs within
1e-3 relative (north_star's fp32 tolerance; bf16 configs feed both sides the
same bf16-rounded values, so the same bound applies). Sizes are chosen so the
oracle finishes in seconds; the benchmarked full-size shapes are in test_gpu_headline.py.
"""
from __future__ import annotations

import numpy as np
import pytest

from tests.helpers import round_bf16, workload

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RTOL = 1e-3  # stated tolerance for fp32 / bf16-input attention outputs


def _dev():
    from paper_2502_08910_b200 import device as D
    D.require_cuda()
    return D


def assert_close(a, b, rtol=RTOL):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    err = np.abs(a - b).max() / max(1e-6, np.abs(b).max())
    assert err <= rtol, f"relative error {err:.3e} > {rtol}"


def run_stage_device(D, stage, lists, q, k, *, n_masks, dtype, layer1=4, stream=0, qstart=0,
                     ext=False, cutoff=3, rope=None, page_size=16):
    """lists: per-mask int arrays (one block). q [H, rows, d]; k [H_kv, T, d]."""
    dev = torch.device("cuda")
    kv = D.PagedKV(torch.from_numpy(k), None, page_size=page_size, dtype=dtype)
    qt = torch.from_numpy(np.ascontiguousarray(q, np.float32)).to(dev)
    stride = max(1, max(len(l) for l in lists))
    in_list = torch.zeros((n_masks, 1, stride), dtype=torch.int32)
    in_count = torch.zeros((n_masks, 1), dtype=torch.int32)
    for m, l in enumerate(lists):
        in_list[m, 0, : len(l)] = torch.from_numpy(np.asarray(l, np.int32))
        in_count[m, 0] = len(l)
    out_list = torch.full((n_masks, 1, max(stride, stage[2])), -7, dtype=torch.int32, device=dev)
    out_count = torch.zeros((n_masks, 1), dtype=torch.int32, device=dev)
    policy = D.RopePolicy(extension=ext, early_cutoff=cutoff)
    D.prune_stage(stage, qt, kv, n_masks=n_masks, in_list=in_list.to(dev), in_count=in_count.to(dev),
                  in_stride=stride, max_chunks=-(-stride // stage[1]), out_list=out_list,
                  out_count=out_count, query_offset=qstart, stream_tokens=stream, layer1=layer1,
                  policy=policy, rope=rope, ws=D.Workspace(dev))
    torch.cuda.synchronize()
    oc = out_count.cpu().numpy()[:, 0]
    ol = out_list.cpu().numpy()[:, 0]
    return [ol[m, : oc[m]] for m in range(n_masks)]


@pytest.mark.parametrize("dtype_name", ["f32", "bf16"])
def test_stage_random_subsets_exact(port, dtype_name):
    """acceptance #6 shapes (acceptance.cpp:220-265): random sorted subsets, random l_c/k."""
    D = _dev()
    dtype = torch.float32 if dtype_name == "f32" else torch.bfloat16
    rng = np.random.default_rng(1006)
    for trial in range(150):
        rows = 1 + rng.integers(3)
        q = rng.standard_normal((1, rows, 8), dtype=np.float32)
        k = rng.standard_normal((1, 96, 8), dtype=np.float32)
        if dtype == torch.bfloat16:
            q, k = round_bf16(q), round_bf16(k)
        idx = np.sort(rng.permutation(96)[: 1 + rng.integers(90)])
        lc = int(1 + rng.integers(8))
        stage = (64, lc, lc * int(1 + rng.integers(8)))
        want = port.run_pruning_stage(stage, idx, q, k)
        got = run_stage_device(D, stage, [idx], q, k, n_masks=1, dtype=dtype)[0]
        assert np.array_equal(got, want), (trial, stage, got, want)
        assert np.all(np.diff(got) > 0)
        assert set(got) <= set(idx)


@pytest.mark.parametrize("ext", [False, True])
def test_stage_rope_policies_exact(port, ext):
    """acceptance #5 setting (acceptance.cpp:146-217): layers 1..6 (chunk-indexed and
    relative), stream 8, random query positions, extension on/off."""
    D = _dev()
    rng = np.random.default_rng(1005)
    rope = D.RopeTable(4096, 8) if ext else None
    for trial in range(120):
        layer1 = int(1 + rng.integers(6))
        qstart = int(rng.integers(2048))
        rows = int(1 + rng.integers(4))
        q = rng.standard_normal((2, rows, 8), dtype=np.float32)
        k = rng.standard_normal((2, 128, 8), dtype=np.float32)
        idx = np.sort(rng.permutation(128)[: 20 + rng.integers(100)])
        lc = int(1 + rng.integers(16))
        stage = (64, lc, lc * int(1 + rng.integers(4)))
        want = port.run_pruning_stage(stage, idx, q, k, layer1=layer1, stream=8, qstart=qstart,
                                      ext=ext, rope_max=4096)
        got = run_stage_device(D, stage, [idx], q, k, n_masks=1, dtype=torch.float32,
                               layer1=layer1, stream=8, qstart=qstart, ext=ext, rope=rope)[0]
        assert np.array_equal(got, want), (trial, layer1, stage)


@pytest.mark.parametrize("dtype_name", ["f32", "bf16"])
@pytest.mark.parametrize("lc", [8, 32, 256])
def test_stage_d128_gqa_exact(port, dtype_name, lc):
    """d=128 fast path, GQA (8 q-heads / 2 kv-heads -> 2 masks of 4), contiguous and
    scattered lists."""
    D = _dev()
    dtype = torch.float32 if dtype_name == "f32" else torch.bfloat16
    q, k, _ = workload(7 + lc, 8, 2, 1, 8192, 128, bf16=dtype == torch.bfloat16)
    rng = np.random.default_rng(lc)
    lists = [np.arange(256, 8192 - 1024, dtype=np.int64),
             np.sort(rng.permutation(np.arange(256, 7168))[:3000])]
    stage = (1, lc, lc * 16)
    got = run_stage_device(D, stage, lists, q, k, n_masks=2, dtype=dtype, qstart=8191, stream=1024,
                           page_size=64)
    for m in range(2):
        want = port.run_pruning_stage(stage, lists[m], q[4 * m: 4 * m + 4], k[m: m + 1],
                                      stream=1024, qstart=8191)
        assert np.array_equal(got[m], want), m


def test_stage_kats(port):
    """test_pruning.cpp:201-235 known answers: identity at budget, needle chunk, constant keys."""
    D = _dev()
    rng = np.random.default_rng(37)
    k = rng.standard_normal((1, 32, 4), dtype=np.float32)
    q = rng.standard_normal((1, 2, 4), dtype=np.float32)
    idx = np.arange(16)
    got = run_stage_device(D, (64, 4, 16), [idx], q, k, n_masks=1, dtype=torch.float32)[0]
    assert np.array_equal(got, idx)  # identity at budget
    k2 = k.copy()
    k2[0, 8:12] = 100.0 * q[0, 0]
    got = run_stage_device(D, (64, 4, 8), [idx], q, k2, n_masks=1, dtype=torch.float32)[0]
    assert len(got) == 8 and {8, 9, 10, 11} <= set(got)
    k3 = np.full_like(k, 0.5)
    got = run_stage_device(D, (64, 4, 8), [idx], q, k3, n_masks=1, dtype=torch.float32)[0]
    assert np.array_equal(got, np.arange(8))  # ties keep the lowest chunks


def _device_build_mask(D, q, k, stages, *, sink, stream, layer0=0, ext=False, n_masks=1,
                       dtype=torch.float32):
    dev = torch.device("cuda")
    kv = D.PagedKV(torch.from_numpy(k), None, page_size=64, dtype=dtype)
    rope = D.RopeTable(k.shape[1] + 2, k.shape[2]) if ext else None
    lists, counts, trace, bs, off = D.build_mask(torch.from_numpy(q).to(dev), kv, stages, sink=sink,
                                                 stream_tokens=stream, layer0=layer0,
                                                 policy=D.RopePolicy(extension=ext), rope=rope,
                                                 n_masks=n_masks)
    torch.cuda.synchronize()
    L = lists.cpu().numpy(); C = counts.cpu().numpy()
    return [[L[m, b, : C[m, b]] for b in range(L.shape[1])] for m in range(n_masks)], bs, off


@pytest.mark.parametrize("ext,layer0", [(False, 0), (True, 0), (True, 4)])
def test_build_mask_multiblock_exact(port, ext, layer0):
    """test_pruning.cpp:323-349 plan: 3 stages with b_q 64 -> 32 -> 16 (sub-block remap)."""
    D = _dev()
    q, k, _ = workload(4, 2, 2, 256, 1024, 16)
    stages = [(64, 16, 256), (32, 8, 128), (16, 4, 64)]
    got, bs, off = _device_build_mask(D, q, k, stages, sink=64, stream=128, layer0=layer0, ext=ext)
    want, _, wbs, woff = port.build_mask(q, k, stages, sink=64, stream=128, layer0=layer0, ext=ext)
    assert (bs, off) == (wbs, woff) == (16, 768)
    assert len(got[0]) == len(want)
    for b, (g, w) in enumerate(zip(got[0], want)):
        assert np.array_equal(g, w), b


def test_build_mask_gqa_bf16_exact(port):
    """GQA masks are per KV group: one oracle call per group."""
    D = _dev()
    q, k, _ = workload(11, 8, 2, 128, 6144, 64, bf16=True)
    stages = [(64, 64, 2048), (64, 16, 512), (64, 4, 128)]
    got, _, _ = _device_build_mask(D, q, k, stages, sink=128, stream=256, n_masks=2,
                                   dtype=torch.bfloat16)
    for m in range(2):
        want, _, _, _ = port.build_mask(q[4 * m: 4 * m + 4], k[m: m + 1], stages, sink=128, stream=256)
        for b in range(len(want)):
            assert np.array_equal(got[m][b], want[b]), (m, b)


@pytest.mark.parametrize("ext", [False, True])
def test_block_sparse_attention_rows(port, ext):
    """BSA over per-row selections (sparse_attention.cpp:114-145), random masks like
    test_sparse_attention.cpp:143-170, within 1e-3 relative."""
    D = _dev()
    dev = torch.device("cuda")
    q, k, v = workload(17, 2, 2, 64, 512, 8)
    rng = np.random.default_rng(21)
    lists = [np.array([i for i in range(16, 416) if rng.integers(4) == 0], np.int32) for _ in range(2)]
    block, sink, stream, off = 32, 16, 32, 512 - 64
    want = port.block_sparse_attention(q, k, v, lists, block_size=block, sink=sink, stream=stream,
                                       offset=off, ext=ext)
    cap = max(len(l) for l in lists)
    ml = torch.zeros((1, 2, cap), dtype=torch.int32)
    mc = torch.zeros((1, 2), dtype=torch.int32)
    for b, l in enumerate(lists):
        ml[0, b, : len(l)] = torch.from_numpy(l)
        mc[0, b] = len(l)
    sel, cnt = D.selected_indices(ml.to(dev), mc.to(dev), n_rows=64, block_size=block,
                                  query_offset=off, sink=sink, stream_tokens=stream)
    # selected lists themselves are index-exact
    for r in (0, 17, 31, 32, 63):
        want_sel = port.selected_indices(lists, block, sink, stream, off, r)
        c = int(cnt[0, r])
        assert np.array_equal(sel[0, r, :c].cpu().numpy(), want_sel)
    kv = D.PagedKV(torch.from_numpy(k), torch.from_numpy(v), page_size=16, dtype=torch.float32)
    rope = D.RopeTable(514, 8) if ext else None
    out = D.bsa(torch.from_numpy(q).to(dev), kv, sel, cnt, query_offset=off, max_sel=sel.shape[-1],
                policy=D.RopePolicy(extension=ext), rope=rope)
    torch.cuda.synchronize()
    assert_close(out.cpu().numpy(), want)


def test_selected_indices_goldens():
    """test_sparse_attention.cpp:181-192 goldens."""
    D = _dev()
    dev = torch.device("cuda")
    ml = torch.tensor([[[2, 5, 7, 11], [2, 5, 7, 11]]], dtype=torch.int32, device=dev)
    mc = torch.tensor([[4, 4]], dtype=torch.int32, device=dev)
    sel, cnt = D.selected_indices(ml, mc, n_rows=8, block_size=4, query_offset=8, sink=2, stream_tokens=3)
    got = lambda r: sel[0, r, : int(cnt[0, r])].cpu().tolist()
    assert got(0) == [0, 1, 2, 5, 6, 7, 8]
    assert got(4) == [0, 1, 2, 5, 7, 10, 11, 12]
    tl = torch.zeros((1, 1, 1), dtype=torch.int32, device=dev)
    tc = torch.zeros((1, 1), dtype=torch.int32, device=dev)
    sel, cnt = D.selected_indices(tl, tc, n_rows=2, block_size=4, query_offset=0, sink=4, stream_tokens=4)
    assert sel[0, 1, : int(cnt[0, 1])].cpu().tolist() == [0, 1]


@pytest.mark.parametrize("case", ["c1_32k_f32", "c1_64k_f32_ext", "gqa_128k_bf16"])
def test_decode_layer_step(port, case):
    """The per-layer decode body (decode.cpp:225-273) with every stage due, 3k preset.
    C1: 32K, 1 head, fp32 (stage 1 is the identity there); a 64K variant exercises
    stage 1; and the Llama GQA shape at 128K in bf16 (2 of the 8 KV groups)."""
    D = _dev()
    dev = torch.device("cuda")
    stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    if case == "c1_32k_f32":
        t, groups, hpm, bf16, ext, layer1 = 32768, 1, 1, False, False, 4
    elif case == "c1_64k_f32_ext":
        t, groups, hpm, bf16, ext, layer1 = 65536, 1, 1, False, True, 2
    else:
        t, groups, hpm, bf16, ext, layer1 = 131072, 2, 4, True, False, 4
    q, k, v = workload(3, groups * hpm, groups, 1, t, 128, bf16=bf16)
    dtype = torch.bfloat16 if bf16 else torch.float32
    kv = D.PagedKV(torch.from_numpy(k), torch.from_numpy(v), page_size=64, dtype=dtype)
    rope = D.RopeTable(t + 2, 128) if ext else None
    layer = D.DecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm,
                          n_masks=groups, layer1=layer1, policy=D.RopePolicy(extension=ext), rope=rope)
    layer.q.copy_(torch.from_numpy(q).to(dev))
    out = layer.run(t).clone()
    torch.cuda.synchronize()
    masks, want_out, _ = port.decode_layer_step(q.reshape(groups, hpm, 128), k, v, stages, sink=256,
                                                stream=1024, ext=ext, layer1=layer1)
    cl, cc = layer.caches[-1]
    for g in range(groups):
        got = cl[g, 0, : int(cc[g, 0])].cpu().numpy()
        assert np.array_equal(got, masks[g]), g
    assert_close(out.cpu().numpy().reshape(groups, hpm, 128), want_out)


@pytest.mark.parametrize("case", ["c1_32k_f32", "c1_64k_f32_ext", "gqa_128k_bf16", "gqa_1m_bf16_g1"])
def test_fused_decode_layer_step(port, case):
    """Fused decode kernels (one kernel per stage, fused top-k, implicit lists, fused
    BSA combine) against the oracle's per-layer decode body."""
    D = _dev()
    dev = torch.device("cuda")
    stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    t, groups, hpm, bf16, ext, layer1 = {
        "c1_32k_f32": (32768, 1, 1, False, False, 4),
        "c1_64k_f32_ext": (65536, 1, 1, False, True, 2),
        "gqa_128k_bf16": (131072, 2, 4, True, False, 4),
        "gqa_1m_bf16_g1": (1 << 20, 1, 4, True, False, 4),
    }[case]
    q, k, v = workload(5, groups * hpm, groups, 1, t, 128, bf16=bf16)
    dtype = torch.bfloat16 if bf16 else torch.float32
    kv = D.PagedKV(torch.from_numpy(k), torch.from_numpy(v), page_size=64, dtype=dtype)
    rope = D.RopeTable(t + 2, 128) if ext else None
    layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm,
                               n_masks=groups, layer1=layer1, policy=D.RopePolicy(extension=ext),
                               rope=rope)
    layer.q.copy_(torch.from_numpy(q[:, 0]).to(dev))
    for _ in range(2):  # second run checks the self-resetting tickets
        out = layer.run(t).clone()
        torch.cuda.synchronize()
        masks, want_out, _ = port.decode_layer_step(q.reshape(groups, hpm, 128), k, v, stages,
                                                    sink=256, stream=1024, ext=ext, layer1=layer1)
        cl, cc = layer.mask()
        for g in range(groups):
            got = cl[g, : int(cc[g])].cpu().numpy()
            assert np.array_equal(got, masks[g]), g
        assert_close(out.cpu().numpy().reshape(groups, hpm, 128), want_out)
    # a step that reuses every cache gathers in the BSA's PDL prologue (mask_stable):
    # same mask, same output (the refresh step may have run on hp_decode_layer, whose
    # split-K partition differs: equal up to fp32 summation order)
    out2 = layer.run(t, refresh=[False] * 3).clone()
    torch.cuda.synchronize()
    assert ((out2 - out).abs().max() / out.abs().max()).item() <= 1e-5


def test_fused_decode_refresh_schedule():
    """Stage caches across steps (decode.cpp:212-249): with intervals (4, 2, 1) the fused
    layer must equal the generic-kernel layer driven by the same refresh flags."""
    D = _dev()
    dev = torch.device("cuda")
    stages = [(1, 64, 4096), (1, 16, 1024), (1, 4, 256)]
    t0, steps, groups, hpm = 40000, 12, 2, 4
    q, k, v = workload(9, groups * hpm, groups, steps, t0 + steps, 128, bf16=True)
    kvf = D.PagedKV(torch.from_numpy(k[:, :t0]), torch.from_numpy(v[:, :t0]), dtype=torch.bfloat16,
                    capacity=t0 + steps)
    kvg = D.PagedKV(torch.from_numpy(k[:, :t0]), torch.from_numpy(v[:, :t0]), dtype=torch.bfloat16,
                    capacity=t0 + steps)
    kw = dict(sink=64, stream_tokens=256, n_q_heads=groups * hpm, n_masks=groups)
    fused = D.FusedDecodeLayer(kvf, stages, **kw)
    generic = D.DecodeLayer(kvg, stages, **kw)
    side = torch.cuda.Stream()
    counters = [0, 0, 0]
    intervals = [4, 2, 1]
    for s in range(steps):
        t = t0 + s + 1
        krow = torch.from_numpy(k[:, t - 1]).to(dev)
        vrow = torch.from_numpy(v[:, t - 1]).to(dev)
        kvf.append(krow, vrow)
        kvg.append(krow, vrow)
        flags = [c == 0 for c in counters]
        qs = torch.from_numpy(q[:, s]).to(dev)
        fused.q.copy_(qs)
        generic.q.copy_(qs.unsqueeze(1))
        of = fused.run(t, refresh=flags, mat_stream=side if s % 2 else None).clone()  # side-branch caches too
        og = generic.run(t, refresh=flags).clone()
        torch.cuda.synchronize()
        for i in range(3):
            fl, fc = fused.mask(i)
            gl, gc = generic.caches[i]
            for g in range(groups):
                n = int(fc[g])
                assert n == int(gc[g, 0])
                assert torch.equal(fl[g, :n].cpu(), gl[g, 0, :n].cpu()), (s, i, g)
        assert_close(of.cpu().numpy(), og[:, 0].cpu().numpy(), rtol=1e-5)
        counters = [(c + 1) % iv for c, iv in zip(counters, intervals)]


def test_fused_step_host_matches_device_path():
    """The host-facing per-layer call (pinned q/K/V in, one H2D copy, append, step with
    side-branch caches, output stored by the kernel into the pinned host buffer) equals the
    device path driven step by step."""
    D = _dev()
    dev = torch.device("cuda")
    stages = [(1, 64, 4096), (1, 16, 1024), (1, 4, 256)]
    t0, steps, groups, hpm = 40000, 4, 2, 4
    q, k, v = workload(13, groups * hpm, groups, steps, t0 + steps, 128, bf16=True)
    kw = dict(sink=64, stream_tokens=256, n_q_heads=groups * hpm, n_masks=groups)
    kv1 = D.PagedKV(torch.from_numpy(k[:, :t0]), torch.from_numpy(v[:, :t0]), dtype=torch.bfloat16,
                    capacity=t0 + steps)
    kv2 = D.PagedKV(torch.from_numpy(k[:, :t0]), torch.from_numpy(v[:, :t0]), dtype=torch.bfloat16,
                    capacity=t0 + steps)
    host = D.FusedDecodeLayer(kv1, stages, **kw)
    ref = D.FusedDecodeLayer(kv2, stages, **kw)
    for s in range(steps):
        t = t0 + s + 1
        flags = [s % 2 == 0, True, s % 2 == 0]
        got = host.step_host(t, q[:, s], k[:, t - 1], v[:, t - 1], refresh=flags).clone()
        kv2.append(torch.from_numpy(k[:, t - 1]).to(dev, torch.bfloat16),
                   torch.from_numpy(v[:, t - 1]).to(dev, torch.bfloat16))
        ref.q.copy_(torch.from_numpy(q[:, s]).to(dev))
        want = ref.run(t, refresh=flags).cpu()
        torch.cuda.synchronize()
        assert torch.equal(got, want), s
        for i in range(3):
            assert torch.equal(host.mask(i)[1], ref.mask(i)[1])


@pytest.mark.parametrize("ext", [False, True])
@pytest.mark.parametrize("t", [1, 7, 300, 1281, 1300, 2049, 5000, 40001])
def test_fused_decode_short_and_ragged_contexts(port, t, ext):
    """Edge contexts on the fused path (3k preset): shorter than the sinks, shorter than
    sink + stream (empty middle), a middle shorter than one stage-1 chunk, ragged last
    pages and chunks — masks exact, outputs within 1e-3 of the oracle's decode body.
    With RoPE extension too (short contexts must not be refused)."""
    D = _dev()
    dev = torch.device("cuda")
    stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    groups, hpm = 2, 4
    q, k, v = workload(17 + t, groups * hpm, groups, 1, t, 128, bf16=True)
    kv = D.PagedKV(torch.from_numpy(k), torch.from_numpy(v), page_size=64, dtype=torch.bfloat16)
    rope = D.RopeTable(t + 2, 128) if ext else None
    layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm,
                               n_masks=groups, policy=D.RopePolicy(extension=ext), rope=rope)
    layer.q.copy_(torch.from_numpy(q[:, 0]).to(dev))
    out = layer.run(t).clone()
    torch.cuda.synchronize()
    masks, want_out, _ = port.decode_layer_step(q.reshape(groups, hpm, 128), k, v, stages, sink=256,
                                                stream=1024, ext=ext, layer1=4)
    cl, cc = layer.mask()
    for g in range(groups):
        assert np.array_equal(cl[g, : int(cc[g])].cpu().numpy(), masks[g]), g
    assert_close(out.cpu().numpy().reshape(groups, hpm, 128), want_out)


def test_descent_reads_the_reference_rows(ref):
    """acceptance #5 (acceptance.cpp:146-217) at 1M: the one-wave stage-1 kernel reads
    exactly as many distinct key rows per KV group as the reference's instrumented
    DirectKeySource (the descent never re-reads a scored row, and it never speculates),
    which is what makes bench.py's row_bits count the algorithmic bytes. The latency-bound
    stages 2/3 deliberately read more (both candidate next rows / whole short chunks)."""
    from paper_2502_08910_b200 import synth
    D = _dev()
    stages = [(64, 256, 32768), (64, 32, 8192), (64, 8, 2048)]
    t, groups, hpm = 1 << 20, 8, 4
    q, k, v = synth.generate(groups * hpm, groups, t, 128, seed=29)
    kv = D.PagedKV(k, v, page_size=64, dtype=torch.bfloat16)
    layer = D.FusedDecodeLayer(kv, stages, sink=256, stream_tokens=1024, n_q_heads=groups * hpm,
                               n_masks=groups)
    layer.q.copy_(q[:, 0])
    layer.run(t)  # materialized caches: each stage below reads its predecessor's list
    torch.cuda.synchronize()
    stride = kv.num_pages * kv.page_size

    def per_group_rows():
        bits = kv.row_bits.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        cnt = torch.zeros_like(bits)
        for sh in range(32):
            cnt += (bits >> sh) & 1
        words = stride // 32
        return [int(cnt[g * words:(g + 1) * words].sum()) for g in range(groups)]

    got = []
    for i in range(3):
        kv.count_rows(True)
        layer.run_stage(t, i, select=False)
        torch.cuda.synchronize()
        got.append(per_group_rows())
        kv.count_rows(False)
    for g in (0, groups - 1):
        want_dis, _ = ref.decode_read_counts(q[g * hpm:(g + 1) * hpm, 0].cpu().numpy(),
                                             k[g].float().cpu().numpy(), stages, sink=256, stream=1024)
        assert got[0][g] == int(want_dis[0]), (g, got[0][g], int(want_dis[0]))
        assert got[1][g] >= int(want_dis[1]) and got[2][g] >= int(want_dis[2])
