"""Memory-safety and race checks of every kernel and variant, without compute-sanitizer.

compute-sanitizer is closed on this GPU pool (profiles/r02/compute_sanitizer_closed.txt), so
each launch is checked by our own means, at reduced sizes:

  * out-of-bounds writes: every output is a view into a larger buffer whose guard bands
    (64 KiB before and after) hold a signalling bit pattern that must survive the call;
  * writes into inputs: the input buffers compare bit-for-bit after the call;
  * races: the call runs three times (with a different unrelated kernel load in between)
    and the outputs must agree bit-for-bit -- a shared-memory or TMEM hand-off race shows
    up as run-to-run differences;
  * every output is finite (uninitialised shared memory or TMEM shows up as NaN/garbage).

Correctness against the oracle is the parity tests' job (test_gpu_parity.py)."""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F, FD, FDD = [("identity",)], [("identity",), ("derivative", 1)], [("identity",), ("derivative", 1), ("derivative", 2)]
GUARD = 16384  # floats (64 KiB) on each side
SENT = 0x7FA5A5A5  # a signalling-NaN bit pattern no kernel writes


def mci():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_10291_b200 as m
    return m


def guarded(shape, dtype):
    """(view, backing): view of `shape` inside a buffer with sentinel guard bands."""
    n = int(np.prod(shape))
    el = torch.empty((), dtype=dtype).element_size()
    words = (n * el + 3) // 4
    back = torch.full((words + 2 * GUARD,), SENT, dtype=torch.int32, device="cuda")
    view = back[GUARD:GUARD + words].view(dtype)[:n].view(*shape)
    return view, back, words


def check_guards(back, words):
    b = back.cpu().numpy()
    assert (b[:GUARD] == SENT).all(), "write before the output buffer"
    assert (b[GUARD + words:] == SENT).all(), "write after the output buffer"


def noise():
    a = torch.randn(1 << 22, device="cuda")
    (a * 1.0001 + 0.5).sum().item()


def run_checked(call, inputs, out_specs):
    """call(outs) -> None; inputs: tensors that must not change; out_specs: [(shape, dtype)]."""
    snap = [x.clone() for x in inputs]
    results = []
    for rep in range(3):
        outs = [guarded(s, d) for s, d in out_specs]
        call([o[0] for o in outs])
        torch.cuda.synchronize()
        for view, back, words in outs:
            check_guards(back, words)
            v = view.cpu()
            vr = torch.view_as_real(v) if v.is_complex() else v
            assert torch.isfinite(vr).all(), "non-finite output"
        results.append([o[0].cpu().clone() for o in outs])
        if rep == 0:
            noise()
    for a, b in zip(inputs, snap):
        assert torch.equal(a, b), "input buffer modified"
    for r in results[1:]:
        for a, b in zip(r, results[0]):
            assert torch.equal(a, b), "run-to-run difference (race?)"


def with_env(monkeypatch, env):
    for k in ("MCI_ROW_VARIANT", "MCI_ROW_QTAB", "MCI_HILBERT_VARIANT", "MCI_DISABLE_ROW", "MCI_LINE_PF",
              "MCI_LINE_VARIANT", "MCI_LINE_TMA", "MCI_LINE_G16", "MCI_LINE_CT8", "MCI_2D_TSTORE", "MCI_2D_ORDER",
              "MCI_2D_STREAMS", "MCI_2D_WS_MB", "MCI_FS_WS_MB", "MCI_FOURSTEP_GENERIC", "MCI_FORCE_ANYLEN",
              "MCI_ROWG"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)


def rnd(shape, dtype=np.float32, seed=0):
    return torch.from_numpy(np.random.default_rng(seed).standard_normal(shape).astype(dtype)).cuda()


CASES_1D = [
    # (id, M, N, L, bank, kwargs, batch, env)
    *[(f"row_v{v}_q{q}", 3, 1024, 16384, FDD, {}, 7, {"MCI_ROW_VARIANT": str(v), "MCI_ROW_QTAB": str(q)})
      for v in range(11) for q in (0, 1)],
    ("row_generic", 3, 1024, 16384, FDD, {}, 5, {"MCI_DISABLE_ROW": "1"}),
    ("rowg_3_1024_ex2", 3, 1024, 16384, FDD, {}, 7, {"MCI_ROWG": "1"}),
    ("rowg_3_1024_deriv", 3, 1024, 16384, FDD, {}, 7, {"MCI_ROWG": "2"}),
    ("rowg_3_1024_table", 3, 1024, 16384, FDD, {}, 7, {"MCI_ROWG": "1", "MCI_ROW_QTAB": "1"}),
    ("rowg_4_1024_deriv", 4, 1024, 16384, FDD + [("derivative", 3)], {}, 7, {}),
    ("rowg_4_1024_delay", 4, 1024, 16384, [("delay", 0.001 * m) for m in range(4)], {}, 7, {}),
    ("rowg_2_2048_deriv", 2, 2048, 16384, FD, {}, 7, {}),
    ("rowg_2_2048_delay", 2, 2048, 16384, [("delay", 0.0), ("delay", 0.0007)], {}, 7, {}),
    ("rowg_8_512_ti", 8, 512, 16384, [("delay", 2 * math.pi * m / 4096) for m in range(8)], {}, 7, {}),
    ("rowg_6_512_table", 6, 512, 16384, [("delay", 0.0003 * m) for m in range(6)], {}, 7, {}),
    ("hilbert_store_wg", 2, 4096, 65536, FD, {"hilbert": True}, 3, {}),
    ("hilbert_direct", 2, 4096, 65536, FD, {"hilbert": True}, 3, {"MCI_HILBERT_VARIANT": "1"}),
    ("hilbert_tma_store", 2, 4096, 65536, FD, {"hilbert": True}, 3, {"MCI_HILBERT_VARIANT": "2"}),
    ("fused_f32", 2, 64, 1024, FD, {}, 9, {}),
    ("fused_f32_hilbert", 2, 64, 1024, FD, {"hilbert": True}, 9, {}),
    ("fused_f64", 2, 64, 1024, FD, {"dtype": "f64"}, 9, {}),
    ("line_pf", 2, 512, 2048, FD, {}, 41, {}),
    ("line_direct", 2, 512, 2048, FD, {}, 41, {"MCI_LINE_PF": "0"}),
    ("line_smem_tables", 2, 512, 2048, FD, {}, 41, {"MCI_LINE_VARIANT": "1"}),
    ("fourstep_fast", 4, 262144, 4194304, [("delay", 2 * math.pi * m / (4 * 262144)) for m in range(4)], {}, 2,
     {"MCI_FS_WS_MB": "64"}),
    ("fourstep_generic", 4, 262144, 4194304, [("delay", 2 * math.pi * m / (4 * 262144)) for m in range(4)], {}, 2,
     {"MCI_FOURSTEP_GENERIC": "1"}),
    ("fourstep_bank", 2, 16384, 131072, FD, {}, 3, {}),
    ("anylen_107", 3, 107, 321, FDD, {}, 9, {}),
    ("anylen_107_hilbert", 3, 107, 321, FDD, {"hilbert": True}, 9, {}),
    ("anylen_107_f64", 3, 107, 321, FDD, {"dtype": "f64"}, 9, {}),
    ("anylen_170", 2, 170, 510, FD, {}, 5, {}),
    ("anylen_forced", 2, 64, 256, FD, {}, 5, {"MCI_FORCE_ANYLEN": "1"}),
]


@pytest.mark.parametrize("cid,M,N,L,bank,kw,batch,env", CASES_1D, ids=[c[0] for c in CASES_1D])
def test_execute_1d_guarded(cid, M, N, L, bank, kw, batch, env, monkeypatch):
    m = mci()
    with_env(monkeypatch, env)
    plan = m.Plan(M, N, L, bank, **kw)
    npdt = np.float64 if kw.get("dtype") == "f64" else np.float32
    g = rnd((batch, M, N), npdt, seed=len(cid))
    tdt = g.dtype
    hil = kw.get("hilbert", False)
    specs = [((batch, L), tdt)] + ([((batch, L), tdt)] if hil else [])

    def call(outs):
        plan.execute(g, *outs)

    run_checked(call, [g], specs)


def test_complex_offgrid_analysis_guarded(monkeypatch):
    m = mci()
    with_env(monkeypatch, {})
    pc = m.Plan(2, 64, 256, [("delay", 0.0), ("delay", 0.01)], complex=True, K1=-10)
    gc = torch.complex(rnd((3, 2, 64), seed=1), rnd((3, 2, 64), seed=2))
    run_checked(lambda o: pc.execute(gc, o[0]), [gc], [((3, 256), torch.complex64)])
    po = m.Plan(3, 107, 321, FDD, offgrid=True, hilbert=True)
    g = rnd((4, 3, 107), seed=3)
    t = torch.from_numpy(np.random.default_rng(4).uniform(-7, 9, 33).astype(np.float32)).cuda()
    run_checked(lambda o: po.execute_offgrid(g, t, o[0], o[1]), [g, t], [((4, 33), torch.float32)] * 2)
    pa = m.Plan(2, 64, 256, FD, analysis=True)
    ga = rnd((5, 2, 64), seed=5)
    run_checked(lambda o: pa.consistency_residual(ga, o[0]), [ga], [((5,), torch.float32)])
    sp = torch.complex(rnd((6, 300), seed=6), rnd((6, 300), seed=7))
    run_checked(lambda o: pa.averaged_error(sp, -150, o[0]), [sp], [((6, 3), torch.float32)])


CASES_2D = [("default", {}), ("g16", {"MCI_LINE_TMA": "0"}), ("g4", {"MCI_LINE_G16": "0"}),
            ("ct8", {"MCI_LINE_CT8": "1"}), ("strided_ws", {"MCI_2D_TSTORE": "0"}), ("rows_first", {"MCI_2D_ORDER": "1"}),
            ("smem_tables", {"MCI_LINE_VARIANT": "1"}), ("two_streams", {"MCI_2D_STREAMS": "2", "MCI_2D_WS_MB": "24"})]


@pytest.mark.parametrize("cid,env", CASES_2D, ids=[c[0] for c in CASES_2D])
def test_execute_2d_guarded(cid, env, monkeypatch):
    m = mci()
    with_env(monkeypatch, env)
    plan = m.Plan2D(2, 512, FD, 2, 512, FD, 4)
    g = rnd((3, 2, 2, 512, 512), seed=11)
    run_checked(lambda o: plan.execute(g, o[0]), [g], [((3, 2048, 2048), torch.float32)])


def test_2d_anylen_and_sisr_guarded(monkeypatch):
    m = mci()
    with_env(monkeypatch, {})
    p = m.Plan2D(2, 60, FD, 2, 56, FD, 3)
    g = rnd((2, 2, 2, 56, 60), seed=12)
    run_checked(lambda o: p.execute(g, o[0]), [g], [((2, 168, 180), torch.float32)])
    s = m.SisrPlan(14, 18, 3)
    lr = rnd((2, 14, 18), seed=13)
    run_checked(lambda o: s.execute(lr, o[0]), [lr], [((2, 42, 54), torch.float32)])
    s64 = m.SisrPlan(20, 20, 4, dtype="f64")
    lr64 = rnd((1, 20, 20), np.float64, seed=14)
    run_checked(lambda o: s64.execute(lr64, o[0]), [lr64], [((1, 80, 80), torch.float64)])
