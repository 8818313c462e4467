"""Pins for oracle/train.py (O9): the hop loop's gradient
against central differences of its own loss on a tiny problem (chain rule
through encoder, residual convolution, halo refresh, decoder and the edge
refresh (iv)); decomposition invariants; SGD / Adam against closed forms."""
import numpy as np
import pytest

from oracle import decomp, train


def _setup(P=1, seed=3, n=40, d=4, k=5, h=2, hid=6):
    g = np.random.default_rng(seed)
    x = g.random((n, 2)).astype(np.float32)
    a = g.normal(size=(n, 1)).astype(np.float32)
    gid = np.arange(n, dtype=np.int64)
    r = 0.35
    l = r * (1 + 2 ** -12)
    _, _, _, ranks = decomp.build_local(x, gid, a, P, l, r, 6, 9, "diff")
    lin = lambda o, i: (g.normal(size=(o, i)) / np.sqrt(i), g.normal(size=o) * 0.1)
    params = dict(enc=[lin(hid, 3), lin(hid, hid), lin(d, hid)],
                  dec=[lin(hid, d), lin(hid, hid), lin(1, hid)],
                  conv=dict(W1=g.normal(size=(k, 3)) * 0.5, b1=g.normal(size=k) * 0.1,
                            W2=g.normal(size=(k, k)) * 0.4, b2=g.normal(size=k) * 0.1,
                            W3=g.normal(size=(d * d, k)) * 0.2, b3=g.normal(size=d * d) * 0.1,
                            b=g.normal(size=d) * 0.1))
    v0 = np.concatenate([x, a], axis=1).astype(np.float64)
    Y = g.normal(size=(n, 1))
    fn = lambda prm, rk=ranks: train.ds_train_grads(prm, rk, lambda rows: v0[rows], lambda rows: Y[rows], h, 2, 1,
                                                    lambda rows: x[rows])
    return params, fn, (x, a, gid, r, l, v0, Y)


def _flat(params):
    out = []
    for part in ("enc", "dec"):
        for l_, (Wl, bl) in enumerate(params[part]):
            out += [(part, l_, 0, Wl), (part, l_, 1, bl)]
    for nm, arr in params["conv"].items():
        out.append(("conv", nm, None, arr))
    return out


def _get(grads, key):
    part, a, b, _ = key
    return grads[part][a][b] if part != "conv" else grads["conv"][a]


def test_train_gradient_central_differences():
    params, fn, _ = _setup()
    loss, grads = fn(params)
    h = 1e-6
    g = np.random.default_rng(0)
    for key in _flat(params):
        arr = key[3]
        gg = _get(grads, key)
        for _ in range(3):  # three random entries per tensor
            idx = tuple(g.integers(0, s) for s in arr.shape)
            old = arr[idx]
            arr[idx] = old + h
            up, _ = fn(params)
            arr[idx] = old - h
            dn, _ = fn(params)
            arr[idx] = old
            num = (up - dn) / (2 * h)
            assert abs(gg[idx] - num) <= 1e-5 * max(1.0, abs(num)), (key[:3], idx, gg[idx], num)


def test_one_hop_decomposed_equals_single_domain():
    # at h = 1 no received value is ever differentiated (the halo latent values
    # are local encoder outputs), so DETACH gives the single-domain gradient
    params, fn1, (x, a, gid, r, l, v0, Y) = _setup(P=1, h=1)
    _, _, _, ranks4 = decomp.build_local(x, gid, a, 4, l, r, 6, 9, "diff")
    l1, g1 = fn1(params)
    l4, g4 = train.ds_train_grads(params, ranks4, lambda rows: v0[rows], lambda rows: Y[rows], 1, 2, 1,
                                  lambda rows: x[rows])
    assert abs(l1 - l4) <= 1e-12 * max(1.0, abs(l1))
    for key in _flat(params):
        assert np.allclose(_get(g1, key), _get(g4, key), rtol=1e-10, atol=1e-12), key[:3]


def test_zero_loss_when_target_is_prediction():
    params, fn, (x, a, gid, r, l, v0, Y) = _setup(h=1)
    _, _, _, ranks = decomp.build_local(x, gid, a, 1, l, r, 6, 9, "diff")
    # the model's own prediction as target
    loss0, _ = fn(params)
    pred = {}

    def Yrows(rows):
        return pred["u"][rows]
    # recompute the prediction with the oracle pieces: one hop, P = 1
    enc_out, _ = train.mlp_fwd(params["enc"], v0[ranks[0]["local_rows"]])
    from oracle import layer as layer_
    out, _ = layer_.layer_fwd(train.conv_desc(3, 4, 5), params["conv"], enc_out, ranks[0]["e"],
                              ranks[0]["row_ptr"], ranks[0]["col_idx"])
    u, _ = train.mlp_fwd(params["dec"], out)
    full = np.zeros((len(v0), 1))
    full[ranks[0]["local_rows"]] = u
    pred["u"] = full
    loss, grads = train.ds_train_grads(params, ranks, lambda rows: v0[rows], Yrows, 1, 2, 1, lambda rows: x[rows])
    assert loss == 0.0
    for key in _flat(params):
        assert np.all(_get(grads, key) == 0.0), key[:3]


def test_sgd_and_adam_closed_forms():
    w = np.array([1.0, -2.0, 3.0])
    g = np.array([0.5, -0.25, 0.0])
    assert np.array_equal(train.sgd(w, g, 0.1), w - 0.1 * g)
    # first Adam step: m_hat = g, v_hat = g^2, so the update is lr * g / (|g| + eps)
    w1, m, v = train.adam(w, g, np.zeros(3), np.zeros(3), 1, 0.01)
    assert np.allclose(w1, w - 0.01 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-15)
    assert np.allclose(m, 0.1 * g) and np.allclose(v, 0.001 * g * g)
