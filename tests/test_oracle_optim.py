"""Pins for oracle/optim.py (O6: P:255; readings R18-R20)."""
import numpy as np
import torch

from oracle import optim as O


def test_adam_matches_torch_optim_adam():
    rng = np.random.default_rng(0)
    theta0 = rng.normal(size=(50, 58))
    lr = O.lr_vector(16, 1e-3, 5e-4, 2.5e-5, 4e-3, 1e-3)
    th = theta0.copy()
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    # torch reference: one Adam per distinct lr group, float64, eps=1e-15
    p = torch.tensor(theta0, dtype=torch.float64, requires_grad=True)
    groups = {}
    for j, l in enumerate(lr):
        groups.setdefault(l, []).append(j)
    params = {l: torch.tensor(theta0[:, js], dtype=torch.float64, requires_grad=True) for l, js in groups.items()}
    opt = torch.optim.Adam([{"params": [params[l]], "lr": l} for l in groups], betas=(0.9, 0.999), eps=1e-15)
    for step in range(1, 6):
        g = rng.normal(size=th.shape) * rng.uniform(1e-4, 1.0)
        th, m, v = O.adam(th, g, m, v, step, lr[None, :])
        opt.zero_grad()
        for l, js in groups.items():
            params[l].grad = torch.tensor(g[:, js], dtype=torch.float64)
        opt.step()
    for l, js in groups.items():
        np.testing.assert_allclose(th[:, js], params[l].detach().numpy(), rtol=1e-12, atol=1e-14)
    _ = p


def test_adam_first_step_is_signed_learning_rate():
    # step 1: m^ = g, v^ = g^2 -> delta = -lr g / (|g| + eps)
    g = np.array([[3.0, -2e-3, 5e-9, 0.0]])
    th, _, _ = O.adam(np.zeros((1, 4)), g, np.zeros((1, 4)), np.zeros((1, 4)), 1, np.array([[1e-3] * 4]))
    np.testing.assert_allclose(th, -1e-3 * g / (np.abs(g) + 1e-15), rtol=1e-12)


def test_reg_gradient_and_eta():
    rng = np.random.default_rng(1)
    S, K = 6, 4
    theta = rng.normal(size=(S, 10 + 3 * K))
    init = theta[:, :10] + rng.normal(size=(S, 10)) * 0.01
    transparent = np.array([True, False, True, False, False, True])
    grad = np.zeros_like(theta)
    grad[1, 12] = 0.5                                        # SH gradient on slot 1 only
    lr = O.lr_vector(K, 1e-3, 5e-4, 2.5e-5, 4e-3, 1e-3)
    eta = np.array([5, 6, 7, 8, 9, 10], dtype=np.int64)
    th2, m2, v2, eta2, gtot = O.unstable_step(theta, grad, np.zeros_like(theta), np.zeros_like(theta), init,
                                              transparent, 1000.0, lr, 1, eta)
    # L_reg = (1/(10 N_t)) sum (theta - theta0)^2 -> central finite differences of that definition
    def Lreg(tg):
        d = (tg - init)[transparent]
        return 1000.0 * (d ** 2).sum() / (10 * transparent.sum())
    h = 1e-6
    for s in range(S):
        for j in range(10):
            tp, tm = theta[:, :10].copy(), theta[:, :10].copy()
            tp[s, j] += h
            tm[s, j] -= h
            fd = (Lreg(tp) - Lreg(tm)) / (2 * h)
            assert abs(gtot[s, j] - fd) < 1e-6 * max(1.0, abs(fd))
    assert list(eta2 - eta) == [0, 1, 0, 0, 0, 0]
    # stable rows of L_reg are untouched, and a zero gradient leaves the parameter in place
    assert np.all(th2[3] == theta[3])


def test_reg_loss_closed_form():
    """L_reg (R18): mean over the 10 N_t geometry scalars of the transparent slots only."""
    import torch

    from oracle.optim import reg_loss
    th = torch.tensor([[1.0] * 10, [2.0] * 10, [5.0] * 10], dtype=torch.float64)
    th0 = torch.zeros_like(th)
    transparent = np.array([True, False, True])
    assert float(reg_loss(th, th0, transparent)) == (10 * 1.0 + 10 * 25.0) / 20
    assert float(reg_loss(th, th0, np.array([False, False, False]))) == 0.0
