"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element, on the same seeded inputs.  Needs a B200 (marker `gpu`)."""
import numpy as np
import pytest

import oracle
import synth
from parity_helpers import check, from_torch_vals, make_case, to_torch_vals

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def geot():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_03019_b200 as g
    return g


def run_reduce(geot, X, idx, S, op, itype="i32", cfg=None, seg_base=0):
    it = torch.int32 if itype == "i32" else torch.int64
    xt = to_torch_vals(X)
    it_ = torch.from_numpy(idx).to(it).cuda()
    y = geot.geot_segment_reduce(xt, it_, S, op, cfg=cfg, seg_base=seg_base)
    torch.cuda.synchronize()
    return from_torch_vals(y)


def parity(geot, E, S, F, op, dtype="f32", mode="real", kind="powerlaw", seed=0, itype="i32", cfg=None):
    if op == "max" and mode == "real":
        mode = "signed"
    L, idx, X = make_case(E, S, F, dtype, mode, kind, seed)
    ref = oracle.segment_reduce(X, idx, S, op, nthreads=oracle.default_threads())
    y = run_reduce(geot, X, idx, S, op, itype, cfg)
    check(y, ref, op, dtype, mode, counts=L, what=f"E={E} S={S} F={F} {op} {dtype} {mode} {kind} {itype} {cfg}")


# ---------------------------------------------------------------- worked examples
@pytest.mark.parametrize("name", ["W1", "W2"])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_worked_examples_gpu(geot, golden, name, op):
    g = golden["worked_examples"]
    x = torch.tensor(g["x"], dtype=torch.float32, device="cuda")
    c = g[name]
    dst = torch.tensor(c["dst"], dtype=torch.int64, device="cuda")
    src = torch.tensor(c["src"], dtype=torch.int64, device="cuda")
    want = np.array(c[op], dtype=np.float32)
    y = geot.index_segment_reduce(src, dst, x, op, num_segments=c["S"]).cpu().numpy()
    np.testing.assert_array_equal(y, want)
    msg = x[src].contiguous()
    y2 = geot.segment_reduce(dst, msg, op, num_segments=c["S"]).cpu().numpy()
    np.testing.assert_array_equal(y2, want)
    off = geot.geot_segment_offsets(dst, c["S"]).cpu().numpy()
    np.testing.assert_array_equal(off, c["offsets"])
    for P, b in c.get("partition", {}).items():
        sb, eb = geot.geot_partition(dst, c["S"], int(P))
        np.testing.assert_array_equal(sb.cpu().numpy(), b["seg"])
        np.testing.assert_array_equal(eb.cpu().numpy(), b["edge"])


# ---------------------------------------------------------------- paper-shaped configs
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
@pytest.mark.parametrize("mode", ["real", "int"])
def test_cora_shaped(geot, op, mode):
    w = synth.workload("cora")
    parity(geot, w["E"], w["S"], w["F"], op, "f32", mode, "powerlaw", w["seed"])


@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_arxiv_shaped_full(geot, op):
    """configs[1] at full size, in the launch configuration bench.py times."""
    w = synth.workload("arxiv")
    parity(geot, w["E"], w["S"], w["F"], op, "f32", "real", "powerlaw", w["seed"])


def test_arxiv_shaped_int_mode(geot):
    w = synth.workload("arxiv")
    parity(geot, w["E"], w["S"], w["F"], "sum", "f32", "int", "powerlaw", w["seed"])


# ---------------------------------------------------------------- widths x skews
WIDTHS = [1, 2, 3, 4, 8, 16, 31, 32, 64, 96, 128, 256, 1024]


@pytest.mark.parametrize("F", WIDTHS)
@pytest.mark.parametrize("kind", ["powerlaw", "uniform", "gaps"])
@pytest.mark.parametrize("mode", ["real", "int"])
def test_widths_sum(geot, F, kind, mode):
    E = 40_000 if F <= 256 else 6_000
    parity(geot, E, E // 9 + 3, F, "sum", "f32", mode, kind, seed=F)


@pytest.mark.parametrize("F", [1, 4, 32, 128, 1024])
@pytest.mark.parametrize("op", ["mean", "max"])
@pytest.mark.parametrize("mode", ["real", "int"])
def test_widths_mean_max(geot, F, op, mode):
    E = 30_000 if F <= 256 else 5_000
    parity(geot, E, E // 7, F, op, "f32", mode, "powerlaw", seed=F + 1)


@pytest.mark.parametrize("kind", synth.STRESS_KINDS)
@pytest.mark.parametrize("op", ["sum", "max"])
def test_stress_families(geot, kind, op):
    parity(geot, 50_000, 3_000, 64, op, "f32", "int", kind, seed=3)


@pytest.mark.parametrize("F", [1, 2, 8, 16, 64, 128, 200, 512])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_bf16(geot, F, op):
    E = 30_000 if F <= 128 else 6_000
    parity(geot, E, E // 11, F, op, "bf16", "real", "powerlaw", seed=F + 2)
    parity(geot, E, E // 11, F, op, "bf16", "int", "powerlaw", seed=F + 3)


@pytest.mark.parametrize("F", [1, 4, 64])
def test_int64_index(geot, F):
    parity(geot, 30_000, 2_000, F, "sum", "f32", "real", "powerlaw", seed=5, itype="i64")
    parity(geot, 30_000, 2_000, F, "max", "f32", "real", "gaps", seed=6, itype="i64")


# ---------------------------------------------------------------- forced configurations
@pytest.mark.parametrize("R", [1, 2, 3, 5, 16, 64])
@pytest.mark.parametrize("vw", [0, 1])
@pytest.mark.parametrize("F", [4, 32, 128])
def test_forced_configs(geot, R, vw, F):
    """Small rows-per-group => many tiles, many carries, middle tiles inside hubs."""
    cfg = {"rows_per_group": R, "vec_elems": vw, "ctas_per_sm": 1}
    for op in ("sum", "mean", "max"):
        parity(geot, 20_000, 700, F, op, "f32", "int", "powerlaw15", seed=R, cfg=cfg)


STREAM = 3  # GEOT_VARIANT_STREAM


@pytest.mark.parametrize("F,dtype", [(16, "f32"), (32, "f32"), (64, "f32"), (96, "f32"), (128, "f32"),
                                     (256, "f32"), (1024, "f32"), (32, "bf16"), (64, "bf16"), (128, "bf16"),
                                     (512, "bf16")])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_stream_variant(geot, F, dtype, op):
    E = 70_000 if F <= 256 else 66_000
    for mode in ("real", "int"):
        parity(geot, E, E // 7, F, op, dtype, mode, "powerlaw15", seed=F, cfg={"variant": STREAM})


# every compiled pipeline (W warps, RS rows per stage, NS stages; NS=1 is the
# LDG register pipeline) of every lane shape (LPR 4/8/16/32, VPL 1..8)
PIPES = {4: [(16, 4, 4), (8, 4, 8), (8, 4, 1)],
         1: [(16, 6, 4), (8, 6, 8), (16, 3, 8), (8, 8, 6), (8, 4, 1), (8, 8, 1), (16, 12, 2), (16, 8, 3)],
         2: [(16, 3, 4), (8, 3, 8), (8, 4, 1)], 4.5: [(8, 3, 4), (8, 2, 1)], 8: [(8, 1, 4), (8, 1, 6), (8, 1, 1)]}


@pytest.mark.parametrize("F,key", [(16, 4), (32, 1), (64, 1), (128, 1), (256, 2), (512, 4.5), (1024, 8)])
def test_stream_every_pipeline(geot, F, key):
    for (w, rs, ns) in PIPES[key]:
        if rs > max(4, min(32, F // 4)) or ((w, rs, ns) in ((16, 12, 2), (16, 8, 3)) and F != 64):
            continue  # (the deeper 16-warp pipelines are compiled for 256-byte rows only)
        cfg = {"variant": STREAM, "warps_per_cta": w, "rows_per_group": rs, "stages": ns}
        for op in ("sum", "max"):
            parity(geot, 90_001, 9_000, F, op, "f32", "int", "powerlaw15", seed=F + w + rs + ns, cfg=cfg)


@pytest.mark.parametrize("kind", synth.STRESS_KINDS)
@pytest.mark.parametrize("F", [16, 32, 128, 512])
def test_stream_stress(geot, kind, F):
    cfg = {"variant": STREAM}
    for op in ("sum", "mean", "max"):
        parity(geot, 100_000, 9_000, F, op, "f32", "int", kind, seed=2, cfg=cfg)


NARROW = 2  # GEOT_VARIANT_NARROW


@pytest.mark.parametrize("F,dtype", [(1, "f32"), (2, "f32"), (4, "f32"), (8, "f32"), (1, "bf16"), (2, "bf16"),
                                     (4, "bf16"), (8, "bf16"), (16, "bf16"),
                                     # lane groups: rows of 64 / 128 bytes as 16-byte lane slices
                                     (16, "f32"), (32, "f32"), (32, "bf16"), (64, "bf16")])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_narrow_variant(geot, F, dtype, op):
    for mode in ("real", "int"):
        parity(geot, 200_003, 200_003 // 9, F, op, dtype, mode, "powerlaw15", seed=F + 7, cfg={"variant": NARROW})


@pytest.mark.parametrize("kind", synth.STRESS_KINDS)
@pytest.mark.parametrize("itype", ["i32", "i64"])
def test_narrow_stress(geot, kind, itype):
    for F in (1, 4, 8, 16, 32):
        for op in ("sum", "mean", "max"):
            parity(geot, 150_001, 12_000, F, op, "f32", "int", kind, seed=5, itype=itype, cfg={"variant": NARROW})


def test_narrow_is_default_for_small_f(geot):
    for F in (1, 2, 4, 8):
        assert geot.geot_select_config(1 << 24, 1 << 20, F, "sum").variant == NARROW
    parity(geot, 1 << 20, 1 << 16, 1, "sum", "f32", "real", "uniform", seed=9)


def test_stream_int64_and_shards(geot):
    parity(geot, 300_000, 20_000, 64, "sum", "f32", "real", "powerlaw", seed=4, itype="i64", cfg={"variant": STREAM})
    L, idx, X = make_case(300_000, 20_000, 128, "f32", "int", "powerlaw15", 5)
    ref = oracle.segment_reduce(X, idx, 20_000, "sum", nthreads=oracle.default_threads())
    xt, it = to_torch_vals(X), torch.from_numpy(idx).to(torch.int32).cuda()
    sb, eb = [b.cpu().numpy() for b in geot.geot_partition(it, 20_000, 3)]
    out = torch.empty((20_000, 128), device="cuda")
    for p in range(3):
        geot.geot_segment_reduce(xt[eb[p]:eb[p + 1]], it[eb[p]:eb[p + 1]], int(sb[p + 1] - sb[p]), "sum",
                                 out=out[sb[p]:sb[p + 1]], seg_base=int(sb[p]), cfg={"variant": STREAM})
    check(out.cpu().numpy(), ref, "sum", "f32", "int", what="stream shards")


def test_stream_is_default_for_arxiv(geot):
    w = synth.workload("arxiv")
    c = geot.geot_select_config(w["E"], w["S"], w["F"], "sum")
    assert c.variant == STREAM


def test_one_hub_across_many_tiles(geot):
    cfg = {"rows_per_group": 1}
    for op in ("sum", "mean", "max"):
        parity(geot, 100_000, 5, 32, op, "f32", "int", "single", seed=1, cfg=cfg)
        parity(geot, 100_000, 5, 32, op, "f32", "real", "single", seed=1)


# ---------------------------------------------------------------- edge cases
def test_empty_and_degenerate(geot):
    # E = 0: every row zero, for every op
    for op in ("sum", "mean", "max"):
        y = geot.geot_segment_reduce(torch.empty((0, 5), device="cuda"), torch.empty(0, dtype=torch.int32,
                                                                                   device="cuda"), 7, op)
        assert y.shape == (7, 5) and torch.all(y == 0) and not torch.any(torch.signbit(y))
    # S = 0
    y = geot.geot_segment_reduce(torch.empty((0, 5), device="cuda"), torch.empty(0, dtype=torch.int32,
                                                                               device="cuda"), 0)
    assert y.shape == (0, 5)
    # single edge, leading and trailing empties
    x = torch.tensor([[2.5, -1.0]], device="cuda")
    y = geot.geot_segment_reduce(x, torch.tensor([3], dtype=torch.int32, device="cuda"), 6, "max").cpu()
    assert torch.equal(y, torch.tensor([[0, 0], [0, 0], [0, 0], [2.5, -1.0], [0, 0], [0, 0]]))


def test_misaligned_pointers_use_scalar_path(geot):
    L, idx, X = make_case(5_000, 400, 32, "f32", "int", "powerlaw", 9)
    big = torch.zeros(X.size + 1, dtype=torch.float32, device="cuda")
    big[1:] = torch.from_numpy(X.ravel()).cuda()
    xt = big[1:].view(X.shape)  # 4-byte aligned only
    assert xt.data_ptr() % 16 != 0
    it = torch.from_numpy(idx).to(torch.int32).cuda()
    ref = oracle.segment_reduce(X, idx, 400, "sum")
    y = geot.geot_segment_reduce(xt, it, 400, "sum")
    check(y.cpu().numpy(), ref, "sum", "f32", "int")


@pytest.mark.parametrize("variant,F,dtype", [(2, 1, "f32"), (2, 4, "f32"), (2, 16, "bf16"), (3, 16, "f32"),
                                             (3, 64, "f32"), (3, 128, "bf16"), (1, 3, "f32"), (1, 64, "f32")])
def test_bad_data_stays_in_bounds(geot, variant, F, dtype):
    """Unsorted keys, keys outside [0, S) and (fused) src ids outside [0, V): results
    are unspecified (P:328 precondition) but every kernel must stay memory-safe —
    no fault, and no store outside `out` (guard rows around it keep their bits)."""
    rng = np.random.default_rng(F + variant)
    # (unsorted keys make every head a "gap" of up to S rows: keep S small, the
    # zero-fill work of garbage input is O(E * S))
    E, S, V, pad = 100_000, 400, 5_000, 64
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    idx = torch.from_numpy(rng.integers(-30, S + 30, E).astype(np.int32)).cuda()
    idx_sorted_bad = torch.sort(idx).values  # sorted, but with out-of-range keys at both ends
    for keys in (idx, idx_sorted_bad):
        big = torch.full((S + 2 * pad, F), 7.0, dtype=tdt, device="cuda")
        X = torch.ones((E, F), dtype=tdt, device="cuda")
        for op in ("sum", "mean", "max"):
            try:
                geot.geot_segment_reduce(X, keys, S, op, out=big[pad:pad + S], cfg={"variant": variant})
            except geot.GeotError as ex:  # a variant may not apply to the shape: that is fine
                assert ex.status == 2, ex
            torch.cuda.synchronize()
            assert torch.all(big[:pad] == 7.0) and torch.all(big[pad + S:] == 7.0), (variant, F, op)
        if variant != 2:  # fused form (no narrow variant)
            x = torch.ones((V, F), dtype=tdt, device="cuda")
            src = torch.from_numpy(rng.integers(-300, V + 300, E).astype(np.int32)).cuda()
            big.fill_(7.0)
            try:
                geot.geot_gather_segment_reduce(x, src, keys, S, "sum", out=big[pad:pad + S], cfg={"variant": variant})
            except geot.GeotError as ex:
                assert ex.status == 2, ex
            torch.cuda.synchronize()
            assert torch.all(big[:pad] == 7.0) and torch.all(big[pad + S:] == 7.0), (variant, F, "fused")


def test_determinism(geot):
    L, idx, X = make_case(200_000, 5_000, 64, "f32", "real", "powerlaw15", 11)
    xt, it = to_torch_vals(X), torch.from_numpy(idx).to(torch.int32).cuda()
    ys = [geot.geot_segment_reduce(xt, it, 5_000, "sum") for _ in range(10)]
    for y in ys[1:]:
        assert torch.equal(y.view(torch.int32), ys[0].view(torch.int32))


# ---------------------------------------------------------------- fused gather (H8)
@pytest.mark.parametrize("F", [1, 16, 64, 128])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_fused_gather(geot, F, op):
    V, E, S = 3_000, 60_000, 2_500
    mode = "signed" if op == "max" else "real"
    L = synth.segment_lengths(E, S, "powerlaw", 4)
    dst = synth.lengths_to_index(L, "i64")
    src = synth.src_index(1004, 0, E, V)
    x = synth.values(4, 0, V, F, "f32", mode)
    ref = oracle.gather_segment_reduce(x, src, dst, S, op, nthreads=oracle.default_threads())
    for it in (torch.int32, torch.int64):
        y = geot.index_segment_reduce(torch.from_numpy(src).to(it).cuda(), torch.from_numpy(dst).to(it).cuda(),
                                      torch.from_numpy(x).cuda(), op, num_segments=S)
        check(y.cpu().numpy(), ref, op, "f32", mode, counts=L, what=f"fused F={F} {op} {it}")


@pytest.mark.parametrize("F", [8, 64])
def test_fused_bf16_and_weighted(geot, F):
    V, E, S = 2_000, 40_000, 1_500
    L = synth.segment_lengths(E, S, "powerlaw", 5)
    dst = synth.lengths_to_index(L, "i64")
    src = synth.src_index(1005, 0, E, V)
    xb = synth.values(5, 0, V, F, "bf16", "real")
    ref = oracle.gather_segment_reduce(xb, src, dst, S, "sum")
    y = geot.index_segment_reduce(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), to_torch_vals(xb),
                                  "sum", num_segments=S)
    check(from_torch_vals(y), ref, "sum", "bf16", "real")
    x = synth.values(6, 0, V, F, "f32", "real")
    w = synth.weights(2006, 0, E)
    refw = oracle.gather_segment_reduce(x, src, dst, S, "sum", weight=w)
    yw = geot.index_weight_segment_reduce(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(),
                                          torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(), num_segments=S)
    check(yw.cpu().numpy(), refw, "sum", "f32", "real")


# -------------------------------------- fused gather through the stream kernel (H8)
def fused_case(E, S, V, F, dtype, mode, kind, seed):
    L = synth.stress_lengths(kind, E, S, seed)
    dst = synth.lengths_to_index(L, "i64")
    src = synth.src_index(seed + 1000, 0, E, V)
    x = synth.values(seed, 0, V, F, dtype, mode)
    return L, dst, src, x


@pytest.mark.parametrize("F,dtype", [(16, "f32"), (32, "f32"), (64, "f32"), (128, "f32"), (32, "bf16"),
                                     (64, "bf16"), (128, "bf16"), (256, "bf16")])
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
def test_fused_gather_stream(geot, F, dtype, op):
    V, E, S = 20_000, 200_003, 15_000
    for mode in (("signed",) if op == "max" else ("int", "real")):
        L, dst, src, x = fused_case(E, S, V, F, dtype, mode, "powerlaw15", F + 3)
        ref = oracle.gather_segment_reduce(x, src, dst, S, op, nthreads=oracle.default_threads())
        for it in (torch.int32, torch.int64):
            y = geot.geot_gather_segment_reduce(to_torch_vals(x), torch.from_numpy(src).to(it).cuda(),
                                                torch.from_numpy(dst).to(it).cuda(), S, op, cfg={"variant": 3})
            check(from_torch_vals(y), ref, op, dtype, mode, counts=L, what=f"gather-stream F={F} {dtype} {op} {it}")


@pytest.mark.parametrize("kind", synth.STRESS_KINDS)
def test_fused_gather_stream_stress_and_weighted(geot, kind):
    V, E, S, F = 9_000, 150_001, 12_000, 64
    for op in ("sum", "mean", "max"):
        L, dst, src, x = fused_case(E, S, V, F, "f32", "int", kind, 6)
        ref = oracle.gather_segment_reduce(x, src, dst, S, op, nthreads=oracle.default_threads())
        for cfg in ({"variant": 3}, {"variant": 3, "warps_per_cta": 16, "rows_per_group": 8, "stages": 3},
                    {"variant": 3, "warps_per_cta": 16, "rows_per_group": 12, "stages": 2}, {"variant": 1}):
            y = geot.geot_gather_segment_reduce(torch.from_numpy(x).cuda(), torch.from_numpy(src).cuda(),
                                                torch.from_numpy(dst).cuda(), S, op, cfg=cfg)
            check(y.cpu().numpy(), ref, op, "f32", "int", counts=L, what=f"gather-stream {kind} {op} {cfg}")
    w = synth.weights(2007, 0, E)
    L, dst, src, x = fused_case(E, S, V, F, "f32", "real", kind, 7)
    refw = oracle.gather_segment_reduce(x, src, dst, S, "sum", weight=w)
    yw = geot.index_weight_segment_reduce(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(),
                                          torch.from_numpy(w).cuda(), torch.from_numpy(x).cuda(), num_segments=S)
    check(yw.cpu().numpy(), refw, "sum", "f32", "real", what=f"weighted gather-stream {kind}")


# every compiled gather pipeline (launch.cuh GEOT_GSHAPE) x weighted / unweighted,
# integer-valued x and weights: bit-exact.  Covers both stage schedules (the
# buffer refilled before the fold when RS <= 8, after it when RS = 12).
GATHER_PIPES = {4: [(16, 4, 4)], 8: [(16, 6, 4), (16, 8, 3)], 16: [(16, 6, 4), (16, 8, 3), (16, 12, 2)],
                32: [(16, 6, 4), (16, 8, 3), (16, 12, 2)]}


@pytest.mark.parametrize("F", [16, 32, 64, 128])
@pytest.mark.parametrize("weighted", [False, True])
def test_gather_every_pipeline(geot, F, weighted):
    V, E, S = 7_000, 180_001, 9_000
    L, dst, src, x = fused_case(E, S, V, F, "f32", "int", "powerlaw15", F + 11)
    w = np.random.default_rng(F).integers(-3, 4, size=E).astype(np.float32) if weighted else None
    ref = oracle.gather_segment_reduce(x, src, dst, S, "sum", weight=w, nthreads=oracle.default_threads())
    lpr = max(4, min(32, F // 4))
    for (W, RS, NS) in GATHER_PIPES[lpr]:
        for it in (torch.int32, torch.int64):
            y = geot.geot_gather_segment_reduce(
                torch.from_numpy(x).cuda(), torch.from_numpy(src).to(it).cuda(), torch.from_numpy(dst).to(it).cuda(),
                S, "sum", weight=None if w is None else torch.from_numpy(w).cuda(),
                cfg={"variant": 3, "warps_per_cta": W, "rows_per_group": RS, "stages": NS})
            check(y.cpu().numpy(), ref, "sum", "f32", "int", counts=L,
                  what=f"gather pipe F={F} ({W},{RS},{NS}) w={weighted} {it}")


# ---------------------------------------------------------------- integer kernels
def test_offsets_partition_validate(geot):
    for kind in synth.STRESS_KINDS:
        L = synth.stress_lengths(kind, 50_000, 4_000, 2)
        idx = synth.lengths_to_index(L, "i64")
        for it in (torch.int32, torch.int64):
            t = torch.from_numpy(idx).to(it).cuda()
            np.testing.assert_array_equal(geot.geot_segment_offsets(t, 4_000).cpu().numpy(),
                                          oracle.offsets(idx, 4_000))
            for P in (1, 2, 3, 4, 8, 13):
                sb, eb = geot.geot_partition(t, 4_000, P)
                osb, oeb = oracle.partition(idx, 4_000, P)
                np.testing.assert_array_equal(sb.cpu().numpy(), osb)
                np.testing.assert_array_equal(eb.cpu().numpy(), oeb)
            assert geot.geot_validate_index(t, 4_000) == oracle.validate(idx, 4_000) == 0
    bad = np.array([0, 3, 2, 9], dtype=np.int64)
    src = np.array([0, 1, 7, 2], dtype=np.int64)
    assert geot.geot_validate_index(torch.from_numpy(bad).cuda(), 5, torch.from_numpy(src).cuda(), 5) == \
        oracle.validate(bad, 5, src, 5) == 7


# ---------------------------------------------------------------- shards (H9 + seg_base)
def test_virtual_shards(geot):
    """Partition, run every shard as an independent call into its slice of out."""
    w = synth.workload("arxiv")
    L = synth.segment_lengths(w["E"], w["S"], "powerlaw", w["seed"])
    idx = synth.lengths_to_index(L, "i64")
    X = synth.values(w["seed"], 0, w["E"], 32, "f32", "int")
    ref = oracle.segment_reduce(X, idx, w["S"], "sum", nthreads=oracle.default_threads())
    xt, it = to_torch_vals(X), torch.from_numpy(idx).to(torch.int32).cuda()
    for P in (2, 3, 8):
        sb, eb = [b.cpu().numpy() for b in geot.geot_partition(it, w["S"], P)]
        out = torch.empty((w["S"], 32), device="cuda")
        for p in range(P):
            geot.geot_segment_reduce(xt[eb[p]:eb[p + 1]], it[eb[p]:eb[p + 1]], int(sb[p + 1] - sb[p]), "sum",
                                     out=out[sb[p]:sb[p + 1]], seg_base=int(sb[p]))
        check(out.cpu().numpy(), ref, "sum", "f32", "int", what=f"P={P}")


# ---------------------------------------------------------------- generator agreement
def test_device_generator_matches_host():
    import synth.device as sd
    for dt, tdt in (("f32", torch.float32), ("bf16", torch.bfloat16)):
        for mode in ("real", "signed", "int"):
            d = sd.values(1000, 24, seed=7, e_begin=123_456, dtype=tdt, mode=mode)
            h = synth.values(7, 123_456, 1000, 24, dt, mode)
            np.testing.assert_array_equal(from_torch_vals(d), h)
    L = synth.segment_lengths(100_000, 7_000, "powerlaw", 3)
    np.testing.assert_array_equal(sd.index_from_lengths(L, torch.int64).cpu().numpy(), synth.lengths_to_index(L))
    np.testing.assert_array_equal(sd.src_index(5000, 977, 1234, e_begin=99).cpu().numpy(),
                                  synth.src_index(1234, 99, 5000, 977))


# ---------------------------------------------------------------- gradients (f3)
@pytest.mark.parametrize("op", ["sum", "mean", "max"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("F", [16, 5])  # 16-byte vectors / the scalar path
def test_segment_reduce_backward(geot, op, dtype, F):
    mode = "int"
    L, idx, X = make_case(30_000, 4_000, F, dtype, mode, "gaps", seed=21)
    rng = np.random.default_rng(3)
    dY = rng.integers(-4, 5, size=(4_000, F)).astype(np.float32)  # exact in bf16 too
    ref = oracle.segment_reduce_backward(dY.astype(np.float64), X, idx, op)
    xt = to_torch_vals(X).requires_grad_(True)
    it = torch.from_numpy(idx).to(torch.int32).cuda()
    y = geot.segment_reduce_autograd(it, xt, op, num_segments=4_000)
    dyt = torch.from_numpy(dY).cuda().to(xt.dtype)
    y.backward(dyt)
    got = xt.grad.float().cpu().numpy().astype(np.float64)
    want = ref
    if dtype == "bf16":  # one RNE rounding of the fp32 gradient
        want = torch.tensor(ref).float().bfloat16().float().numpy().astype(np.float64)
    elif op != "sum":
        want = ref.astype(np.float32).astype(np.float64)  # fp32 division, one rounding
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("op", ["sum", "mean"])
@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("F", [32, 6])  # vector reductions / the scalar path
def test_gather_backward_and_sddmm(geot, op, weighted, F):
    V, E, S = 1_000, 20_000, 800
    L = synth.segment_lengths(E, S, "powerlaw", 8)
    dst = synth.lengths_to_index(L, "i64")
    src = synth.src_index(1008, 0, E, V)
    x = synth.values(8, 0, V, F, "f32", "int")
    w = (np.random.default_rng(1).integers(1, 4, size=E).astype(np.float32)) if weighted else None
    dY = np.random.default_rng(2).integers(-3, 4, size=(S, F)).astype(np.float64)
    dx_ref, dw_ref = oracle.gather_segment_reduce_backward(dY, x, src, dst, op, weight=w)
    xt = torch.from_numpy(x).cuda().requires_grad_(True)
    wt = torch.from_numpy(w).cuda().requires_grad_(True) if weighted else None
    srct, dstt = torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda()
    if weighted and op == "mean":
        pytest.skip("weighted form is sum-only (P:330)")
    y = geot.index_segment_reduce_autograd(srct, dstt, xt, op, weight=wt, num_segments=S)
    y.backward(torch.from_numpy(dY).float().cuda())
    gx = xt.grad.cpu().numpy().astype(np.float64)
    if op == "sum":  # integer-valued terms: every fp32 partial sum is exact => bit-exact
        np.testing.assert_array_equal(gx, dx_ref)
    else:
        # R14 rule: |dx - dx64| <= 1e-5 * sum over the scattered terms of |w g dY|
        # (tolerance denominator by numpy, from the same inputs)
        counts = np.bincount(dst, minlength=S).astype(np.float64)
        term = np.abs(dY[dst] / counts[dst][:, None] * (1.0 if w is None else np.abs(w)[:, None]))
        A = np.zeros_like(dx_ref)
        np.add.at(A, src, term)
        assert np.all(np.abs(gx - dx_ref) <= 1e-5 * A)
    if weighted:
        g = np.ones(E) if op == "sum" else 1.0 / np.bincount(dst, minlength=S)[dst]
        Aw = g * np.abs(x[src].astype(np.float64) * dY[dst]).sum(axis=1)
        assert np.all(np.abs(wt.grad.cpu().numpy().astype(np.float64) - dw_ref) <= 1e-5 * Aw)


# ---------------------------------------------------------------- workspace poisoning
@pytest.mark.timeout(300)
@pytest.mark.parametrize("F,variant", [(128, 3), (1, 2)])
def test_poisoned_workspace_recovers(geot, F, variant):
    """A workspace whose control words are not at rest (here: a stale ticket)
    must neither hang nor trap: the call retires, geot_workspace_status reports
    the poison, and checked=True repairs the workspace and recomputes."""
    E, S = 400_000, 30_000
    L, idx, X = make_case(E, S, F, "f32", "int", "powerlaw", seed=12)
    ref = oracle.segment_reduce(X, idx, S, "sum", nthreads=oracle.default_threads())
    xt, it = to_torch_vals(X), torch.from_numpy(idx).to(torch.int32).cuda()
    cfg = {"variant": variant}
    geot.geot_segment_reduce(xt, it, S, "sum", cfg=cfg)
    torch.cuda.synchronize()
    key = (xt.device, torch.cuda.current_stream().cuda_stream)
    assert geot.geot_workspace_check(repair=False)[key] == 0
    geot._ws_cache[key].view(torch.int32)[0] = 7  # the ticket word of the control block
    geot.geot_segment_reduce(xt, it, S, "sum", cfg=cfg)  # retires without output; must return
    torch.cuda.synchronize()
    assert geot.geot_workspace_check(repair=False)[key] & 1
    y = geot.geot_segment_reduce(xt, it, S, "sum", cfg=cfg, checked=True)
    torch.cuda.synchronize()
    check(from_torch_vals(y), ref, "sum", "f32", "int", what="after repair")
    assert geot.geot_workspace_check(repair=False)[key] == 0
