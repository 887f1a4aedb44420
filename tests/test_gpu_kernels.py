"""Kernel-level parity on the B200: the tcgen05 GEMM with every fused epilogue and the
flash attention kernel, each against a plain PyTorch fp32 reference of the same op on the
same bf16 inputs (the op semantics are the reference's, proj/src/evaluate.cpp:160-252)."""
import math

import numpy as np
import pytest
import torch

from paper_2510_26742_b200 import engine as E

pytestmark = pytest.mark.gpu

dev = "cuda"


def _ptr(t):
    return None if t is None else t.data_ptr()


def _run_gemm(A, W, mode, flags=0, *, N=None, bn=128, splits=1, row_stats=None, inv_width=0.0, bias=None,
              table_row=None, rope_cs=None, rope_pos0=0, rope_cols=0, resid_scale=1.0, out=None, outb=None,
              out_stats=None, row0_src=None, ld_out=None):
    M, K = A.shape
    N = N or W.shape[0]
    ws = torch.zeros(max(1, M * N), dtype=torch.float32, device=dev)
    ctr = torch.zeros(4096, dtype=torch.int32, device=dev)
    d = E.GemmDesc()
    d.a, d.lda = A.data_ptr(), A.stride(0)
    d.w, d.ldw = W.data_ptr(), W.stride(0)
    d.M, d.N, d.K = M, N, K
    d.bn, d.splits, d.mode, d.flags = bn, splits, mode, flags
    d.row_stats, d.inv_width, d.eps = _ptr(row_stats), inv_width, 1e-6
    d.bias, d.table_row = _ptr(bias), _ptr(table_row)
    d.rope_cs, d.rope_pos0, d.rope_cols = _ptr(rope_cs), rope_pos0, rope_cols
    d.resid_scale = resid_scale
    d.out, d.ldo = out.data_ptr(), ld_out or out.stride(0)
    d.outb, d.ldob = _ptr(outb), (outb.stride(0) if outb is not None else 0)
    d.out_stats, d.row0_src = _ptr(out_stats), _ptr(row0_src)
    d.ws, d.counters = ws.data_ptr(), ctr.data_ptr()
    E.gemm(d)
    torch.cuda.synchronize()
    assert float(ws.abs().max()) == 0.0, "split-K workspace not left clean"
    assert int(ctr.abs().max()) == 0, "split-K counters not reset"


def _rand(shape, scale=1.0, dtype=torch.bfloat16, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    return (torch.rand(shape, generator=g, device=dev, dtype=torch.float32) * 2 - 1).mul_(scale).to(dtype)


def _close(got, ref, rtol):
    got = got.float()
    ref = ref.float()
    scale = ref.abs().max().item() + 1e-12
    err = (got - ref).abs().max().item() / scale
    assert err < rtol, f"max err {err:.3e} (rel to max {scale:.3e}) >= {rtol}"


def _rope_table(npos):
    j = torch.arange(128, dtype=torch.float64)
    freq = torch.pow(torch.tensor(10000.0, dtype=torch.float64), -2.0 * j / 256.0)
    ang = torch.arange(npos, dtype=torch.float64)[:, None] * freq[None, :]
    return torch.stack([ang.cos(), ang.sin()], dim=-1).float().contiguous().to(dev)


@pytest.mark.parametrize("M,N,K,bn,splits", [
    (512, 1152, 1152, 128, 1), (512, 1152, 1152, 128, 4), (256, 4304, 1152, 128, 1),
    (64, 2560, 1024, 256, 8), (63, 1024, 32, 128, 1), (1, 1024, 32, 128, 1), (512, 1152, 588, 128, 1),
    (300, 256, 640, 64, 3),
])
def test_gemm_bf16_rowscale_bias(M, N, K, bn, splits):
    A = _rand((M, (K + 7) // 8 * 8), seed=1)[:, :K]   # TMA needs a 16-byte row pitch
    W = _rand((N, (K + 7) // 8 * 8), 1 / math.sqrt(K), seed=2)[:, :K]
    stats = torch.rand(M, device=dev) * K + 1.0
    bias = _rand((N,), 0.1, torch.float32, seed=3)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_gemm(A, W, E.MODE_BF16, E.FLAG_ROWSCALE | E.FLAG_BIAS, bn=bn, splits=splits, row_stats=stats,
              inv_width=1.0 / K, bias=bias, out=out)
    s = 1.0 / torch.sqrt(stats / K + 1e-6)
    ref = (A.float() @ W.float().T) * s[:, None] + bias[None, :]
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("splits", [1, 2])
def test_gemm_gelu(splits):
    M, N, K = 512, 4304, 1152
    A, W = _rand((M, K), seed=4), _rand((N, K), 1 / math.sqrt(K), seed=5)
    bias = _rand((N,), 0.1, torch.float32, seed=6)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_gemm(A, W, E.MODE_BF16, E.FLAG_BIAS | E.FLAG_GELU, bn=128, splits=splits, bias=bias, out=out)
    ref = torch.nn.functional.gelu(A.float() @ W.float().T + bias, approximate="tanh")
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("M,splits,pos0", [(512, 1, 0), (512, 3, 0), (64, 8, 512), (800, 1, 0)])
def test_gemm_rope(M, splits, pos0):
    K, q, kv = 2048, 2048, 256
    N = q + 2 * kv
    A, W = _rand((M, K), seed=7), _rand((N, K), 1 / math.sqrt(K), seed=8)
    stats = torch.rand(M, device=dev) * K + 1.0
    cs = _rope_table(pos0 + M)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_gemm(A, W, E.MODE_BF16, E.FLAG_ROWSCALE | E.FLAG_ROPE, bn=256, splits=splits, row_stats=stats,
              inv_width=1.0 / K, rope_cs=cs, rope_pos0=pos0, rope_cols=q + kv, out=out)
    z = (A.float() @ W.float().T) / torch.sqrt(stats / K + 1e-6)[:, None]
    c = cs[pos0:pos0 + M, :, 0]
    s = cs[pos0:pos0 + M, :, 1]
    ref = z.clone()
    for h0 in range(0, q + kv, 256):
        a, b = z[:, h0:h0 + 128], z[:, h0 + 128:h0 + 256]
        ref[:, h0:h0 + 128] = a * c - b * s
        ref[:, h0 + 128:h0 + 256] = a * s + b * c
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("M,mlp,K,splits", [(512, 1024, 512, 1), (64, 4096, 1024, 4), (64, 512, 256, 2)])
def test_gemm_gate(M, mlp, K, splits):
    A = _rand((M, K), seed=9)
    Wlog = _rand((2 * mlp, K), 1 / math.sqrt(K), seed=10)   # logical [up | gate] rows
    # pack: tile t = up[128t:128t+128] then gate[128t:128t+128] (csrc/kernels_misc.cu packed_row)
    up, gate = Wlog[:mlp], Wlog[mlp:]
    Wp = torch.stack([up.view(mlp // 128, 128, K), gate.view(mlp // 128, 128, K)], 1).reshape(2 * mlp, K)
    stats = torch.rand(M, device=dev) * K + 1.0
    out = torch.zeros(M, mlp, dtype=torch.bfloat16, device=dev)
    _run_gemm(A, Wp.contiguous(), E.MODE_GATE, E.FLAG_ROWSCALE, N=2 * mlp, bn=256, splits=splits,
              row_stats=stats, inv_width=1.0 / K, out=out)
    z = (A.float() @ Wlog.float().T) / torch.sqrt(stats / K + 1e-6)[:, None]
    ref = z[:, :mlp] * torch.nn.functional.gelu(z[:, mlp:], approximate="tanh")
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("M,N,K,bn,splits,scale,flags", [
    (512, 1152, 1152, 128, 1, 1.0, 2), (512, 1152, 4304, 128, 4, 1.0, 2), (512, 2048, 16384, 256, 4, 1.0, 0),
    (64, 1024, 4096, 128, 16, 1.0, 0), (63, 32, 1024, 64, 1, 0.1, 3), (63, 32, 1024, 64, 4, 0.1, 3),
])
def test_gemm_residual(M, N, K, bn, splits, scale, flags):
    A, W = _rand((M, K), seed=11), _rand((N, K), 1 / math.sqrt(K), seed=12)
    h0 = _rand((M, N), 1.0, torch.float32, seed=13)
    h = h0.clone()
    hb = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    st = torch.zeros(M, device=dev)
    stats = torch.rand(M, device=dev) * K + 1.0
    bias = _rand((N,), 0.1, torch.float32, seed=14)
    _run_gemm(A, W, E.MODE_RESID, flags, bn=bn, splits=splits, row_stats=stats, inv_width=1.0 / K, bias=bias,
              resid_scale=scale, out=h, outb=hb, out_stats=st)
    z = A.float() @ W.float().T
    if flags & E.FLAG_ROWSCALE:
        z = z / torch.sqrt(stats / K + 1e-6)[:, None]
    if flags & E.FLAG_BIAS:
        z = z + bias
    ref = h0 + scale * z
    _close(h, ref, 2e-5 * max(1.0, K / 1024))
    _close(hb, ref, 1e-2)
    _close(st, (ref * ref).sum(1), 1e-4)


@pytest.mark.parametrize("splits", [1, 4])
def test_gemm_f32_store_row0(splits):
    M, N, K = 63, 1024, 1024
    A, W = _rand((M, K), seed=15), _rand((N, K), 1 / math.sqrt(K), seed=16)
    bias = _rand((N,), 0.1, torch.float32, seed=17)
    row0 = _rand((N,), 1.0, torch.float32, seed=18)
    y = torch.zeros(M + 1, N, device=dev)
    yb = torch.zeros(M + 1, N, dtype=torch.bfloat16, device=dev)
    st = torch.zeros(M + 1, device=dev)
    d_out = y[1:]
    _run_gemm(A, W, E.MODE_F32_STORE, E.FLAG_BIAS, bn=128, splits=splits, bias=bias, out=d_out, outb=yb[1:],
              out_stats=st[1:], row0_src=row0)
    ref = torch.cat([row0[None], A.float() @ W.float().T + bias], 0)
    _close(y, ref, 2e-5)
    _close(yb, ref, 1e-2)
    _close(st, (ref * ref).sum(1), 1e-4)


def test_gemm_silu_table():
    M, N, K = 63, 1024, 32
    A, W = _rand((M, K), seed=19), _rand((N, K), 1 / math.sqrt(K), seed=20)
    tab = _rand((N,), 0.2, torch.float32, seed=21)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_gemm(A, W, E.MODE_SILU_TABLE, 0, bn=128, table_row=tab, out=out)
    ref = torch.nn.functional.silu(A.float() @ W.float().T + tab)
    _close(out, ref, 1e-2)


# ------------------------------------------------------------------ attention

def _attn_ref(q, k, v, heads, kv_heads, hd):
    rows = q.shape[0]
    out = torch.zeros(rows, heads * hd, device=dev)
    for h in range(heads):
        kvh = h % kv_heads
        qh = q[:, h * hd:(h + 1) * hd].float()
        kh = k[:, kvh * hd:(kvh + 1) * hd].float()
        vh = v[:, kvh * hd:(kvh + 1) * hd].float()
        p = torch.softmax(qh @ kh.T / math.sqrt(hd), dim=-1)
        out[:, h * hd:(h + 1) * hd] = p @ vh
    return out


@pytest.mark.parametrize("hd,heads,kv_heads,q_rows,rows0,rows1,splits,rows0_valid", [
    (72, 16, 16, 512, 512, 0, 0, 0), (72, 16, 16, 768, 768, 0, 0, 0), (72, 4, 4, 256, 256, 0, 2, 0),
    (256, 8, 1, 512, 512, 0, 0, 0), (256, 8, 1, 800, 800, 0, 0, 0), (256, 8, 1, 512, 512, 0, 1, 0),
    (256, 8, 1, 64, 512, 64, 0, 0), (256, 8, 1, 64, 800, 64, 0, 0), (256, 2, 1, 64, 256, 64, 4, 0),
    (72, 16, 16, 512, 512, 0, 2, 0), (256, 8, 1, 512, 512, 0, 4, 0), (256, 8, 1, 800, 800, 0, 8, 0),
    (72, 16, 16, 768, 768, 0, 8, 0),
    # unaligned prefixes (any prompt length): one segment of 557 keys read in 64-row boxes with the
    # rows past it zero-filled and masked; and a 32-aligned segment of 576 rows whose last 19 are
    # padding (rows0_valid) ahead of the action expert's own 64 keys
    (256, 8, 1, 576, 557, 0, 0, 0), (256, 8, 1, 576, 557, 0, 4, 0), (72, 16, 16, 288, 275, 0, 0, 0),
    (256, 8, 1, 64, 576, 64, 0, 557), (256, 2, 1, 64, 800, 64, 2, 775),
])
def test_attention(hd, heads, kv_heads, q_rows, rows0, rows1, splits, rows0_valid):
    # q/k/v live in one qkv-style buffer like the engine's (row stride = q + 2 kv)
    qw, kvw = heads * hd, kv_heads * hd
    ld = qw + 2 * kvw
    X = _rand((max(q_rows, rows0), ld), 2.0, seed=22)
    Y = _rand((max(rows1, 1), ld), 2.0, seed=23)
    q = X[:q_rows, :qw] if rows1 == 0 else Y[:q_rows, :qw]
    if rows1:
        Y = _rand((q_rows, ld), 2.0, seed=24)
        q = Y[:, :qw]
    k0, v0 = X[:rows0, qw:qw + kvw], X[:rows0, qw + kvw:]
    out = torch.zeros(q_rows, qw, dtype=torch.bfloat16, device=dev)
    d = E.AttnDesc()
    d.head_dim = hd
    d.q, d.ldq, d.q_rows, d.heads, d.kv_heads = q.data_ptr(), ld, q_rows, heads, kv_heads
    d.k0, d.v0, d.ld0, d.rows0 = k0.data_ptr(), v0.data_ptr(), ld, rows0
    if rows1:
        d.k1, d.v1, d.ld1, d.rows1 = Y[:, qw:qw + kvw].data_ptr(), Y[:, qw + kvw:].data_ptr(), ld, rows1
    d.out, d.ldo = out.data_ptr(), qw
    d.kv_splits = splits
    d.rows0_valid = rows0_valid
    n_ws = E.attention_ws_floats(d)
    ws = torch.zeros(max(1, n_ws), device=dev)
    ctr = torch.zeros(4096, dtype=torch.int32, device=dev)
    d.ws, d.counters = ws.data_ptr(), ctr.data_ptr()
    E.attention(d)
    torch.cuda.synchronize()
    n0 = rows0_valid or rows0  # padding keys of segment 0 take no part
    if rows1:
        kk = torch.cat([k0[:n0], Y[:, qw:qw + kvw]], 0)
        vv = torch.cat([v0[:n0], Y[:, qw + kvw:]], 0)
    else:
        kk, vv = k0[:n0], v0[:n0]
    ref = _attn_ref(q, kk, vv, heads, kv_heads, hd)
    _close(out, ref, 2e-2)
    assert int(ctr.abs().max()) == 0


# ------------------------------------------------------------------ skinny (action expert) GEMM

def _pack_rows(perm, m, rope_cols=0):
    """packed row index of every logical column (csrc/kernels_misc.cu packed_row)."""
    j = np.arange(m)
    if perm == E.PERM_GATE64:
        half = m // 2
        gate = j >= half
        c = np.where(gate, j - half, j)
        return (c // 64) * 128 + np.where(gate, 64, 0) + c % 64
    if perm == E.PERM_ROPE:
        h, w = j >> 8, j & 255
        part, i = w >> 7, w & 127
        r = (h << 8) + (i >> 6) * 128 + part * 64 + (i & 63)
        return np.where(j < rope_cols, r, j)
    return j


def _run_skinny(X, Wlog, mode, flags=0, *, perm=E.PERM_NONE, cluster=1, row_stats=None, bias=None, table_row=None,
                rope_cs=None, rope_pos0=0, rope_cols=0, resid_scale=1.0, out=None, outb=None, out_stats=None,
                row0_src=None):
    M, K = X.shape
    N = Wlog.shape[0]
    rows = torch.as_tensor(_pack_rows(perm, N, rope_cols), device=dev)
    Wp = torch.empty_like(Wlog)
    Wp[rows] = Wlog
    d = E.GemmDesc()
    d.a, d.lda = X.data_ptr(), X.stride(0)
    d.w, d.ldw = Wp.data_ptr(), Wp.stride(0)
    d.M, d.N, d.K = M, N, K
    d.mode, d.flags = mode, flags
    d.row_stats, d.inv_width, d.eps = _ptr(row_stats), 1.0 / K, 1e-6
    d.bias, d.table_row = _ptr(bias), _ptr(table_row)
    d.rope_cs, d.rope_pos0, d.rope_cols = _ptr(rope_cs), rope_pos0, rope_cols
    d.resid_scale = resid_scale
    d.out, d.ldo = out.data_ptr(), out.stride(0)
    d.outb, d.ldob = _ptr(outb), (outb.stride(0) if outb is not None else 0)
    d.out_stats, d.row0_src = _ptr(out_stats), _ptr(row0_src)
    E.gemm_skinny(d, cluster)
    torch.cuda.synchronize()


@pytest.mark.parametrize("M,N,K,cluster", [(64, 1024, 2048, 8), (63, 1024, 1024, 4), (1, 1024, 32, 1),
                                           (64, 384, 640, 2), (64, 32, 1024, 8)])
def test_skinny_plain(M, N, K, cluster):
    X, W = _rand((M, K), seed=31), _rand((N, K), 1 / math.sqrt(K), seed=32)
    stats = torch.rand(M, device=dev) * K + 1.0
    bias = _rand((N,), 0.1, torch.float32, seed=33)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_skinny(X, W, E.MODE_BF16, E.FLAG_ROWSCALE | E.FLAG_BIAS, cluster=cluster, row_stats=stats, bias=bias, out=out)
    ref = (X.float() @ W.float().T) / torch.sqrt(stats / K + 1e-6)[:, None] + bias
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("cluster", [1, 4, 8])
def test_skinny_rope(cluster):
    M, K, q, kv = 64, 1024, 2048, 256
    N = q + 2 * kv
    X, W = _rand((M, K), seed=34), _rand((N, K), 1 / math.sqrt(K), seed=35)
    stats = torch.rand(M, device=dev) * K + 1.0
    pos0 = 512
    cs = _rope_table(pos0 + M)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_skinny(X, W, E.MODE_BF16, E.FLAG_ROWSCALE | E.FLAG_ROPE, perm=E.PERM_ROPE, cluster=cluster, row_stats=stats,
                rope_cs=cs, rope_pos0=pos0, rope_cols=q + kv, out=out)
    z = (X.float() @ W.float().T) / torch.sqrt(stats / K + 1e-6)[:, None]
    c, s = cs[pos0:pos0 + M, :, 0], cs[pos0:pos0 + M, :, 1]
    ref = z.clone()
    for h0 in range(0, q + kv, 256):
        a, b = z[:, h0:h0 + 128], z[:, h0 + 128:h0 + 256]
        ref[:, h0:h0 + 128] = a * c - b * s
        ref[:, h0 + 128:h0 + 256] = a * s + b * c
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("mlp,cluster", [(4096, 2), (512, 1), (512, 8)])
def test_skinny_gate(mlp, cluster):
    M, K = 64, 1024
    X, W = _rand((M, K), seed=36), _rand((2 * mlp, K), 1 / math.sqrt(K), seed=37)
    stats = torch.rand(M, device=dev) * K + 1.0
    out = torch.zeros(M, mlp, dtype=torch.bfloat16, device=dev)
    _run_skinny(X, W, E.MODE_GATE, E.FLAG_ROWSCALE, perm=E.PERM_GATE64, cluster=cluster, row_stats=stats, out=out)
    z = (X.float() @ W.float().T) / torch.sqrt(stats / K + 1e-6)[:, None]
    ref = z[:, :mlp] * torch.nn.functional.gelu(z[:, mlp:], approximate="tanh")
    _close(out, ref, 1e-2)


@pytest.mark.parametrize("M,N,K,cluster,scale,flags", [(64, 1024, 4096, 8, 1.0, 0), (64, 1024, 2048, 1, 1.0, 0),
                                                       (63, 32, 1024, 8, 0.1, 3)])
def test_skinny_residual(M, N, K, cluster, scale, flags):
    X, W = _rand((M, K), seed=38), _rand((N, K), 1 / math.sqrt(K), seed=39)
    h0 = _rand((M, N), 1.0, torch.float32, seed=40)
    h = h0.clone()
    hb = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    st = torch.zeros(M, device=dev)
    stats = torch.rand(M, device=dev) * K + 1.0
    bias = _rand((N,), 0.1, torch.float32, seed=41)
    _run_skinny(X, W, E.MODE_RESID, flags, cluster=cluster, row_stats=stats, bias=bias, resid_scale=scale, out=h,
                outb=hb, out_stats=st)
    z = X.float() @ W.float().T
    if flags & E.FLAG_ROWSCALE:
        z = z / torch.sqrt(stats / K + 1e-6)[:, None]
    if flags & E.FLAG_BIAS:
        z = z + bias
    ref = h0 + scale * z
    _close(h, ref, 2e-5 * max(1.0, K / 1024))
    _close(hb, ref, 1e-2)
    _close(st, (ref * ref).sum(1), 1e-4)


@pytest.mark.parametrize("cluster", [1, 8])
def test_skinny_f32_store_row0_and_silu(cluster):
    M, N, K = 63, 1024, 1024
    X, W = _rand((M, K), seed=42), _rand((N, K), 1 / math.sqrt(K), seed=43)
    bias = _rand((N,), 0.1, torch.float32, seed=44)
    row0 = _rand((N,), 1.0, torch.float32, seed=45)
    y = torch.zeros(M + 1, N, device=dev)
    yb = torch.zeros(M + 1, N, dtype=torch.bfloat16, device=dev)
    st = torch.zeros(M + 1, device=dev)
    _run_skinny(X, W, E.MODE_F32_STORE, E.FLAG_BIAS, cluster=cluster, bias=bias, out=y[1:], outb=yb[1:],
                out_stats=st[1:], row0_src=row0)
    ref = torch.cat([row0[None], X.float() @ W.float().T + bias], 0)
    _close(y, ref, 2e-5)
    _close(yb, ref, 1e-2)
    _close(st, (ref * ref).sum(1), 1e-4)
    Xs, Ws = _rand((M, 32), seed=46), _rand((N, 32), 1 / math.sqrt(32), seed=47)
    tab = _rand((N,), 0.2, torch.float32, seed=48)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device=dev)
    _run_skinny(Xs, Ws, E.MODE_SILU_TABLE, 0, cluster=1, table_row=tab, out=out)
    _close(out, torch.nn.functional.silu(Xs.float() @ Ws.float().T + tab), 1e-2)
