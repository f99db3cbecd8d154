"""-m "not gpu": the algebra behind the GPU path's nu = 2 inner-FCG "z-form".

The library's fcg_inner (driver.cu) does not form the second direction d_1 = z - beta_0 d_0 or
q_1 = A d_1.  From one pass over z it takes z.Az, z.q_0 and z.rho_1 and uses
  beta_0 = z.q_0 / d_0.q_0,   d_1.q_1 = z.Az - beta_0 z.q_0,   d_1.rho_1 = z.rho_1,
  E = (alpha_0 - alpha_1 beta_0) d_0 + alpha_1 z.
That is the flexible CG step of PAPER.md l.321 only because A is symmetric
(d_0.Az = q_0.z) and alpha_0 makes rho_1 orthogonal to d_0.  These tests check the identity against
the direct two-step FCG written out in numpy, for an arbitrary (nonlinear) preconditioner output z,
and the A13 guards (zero denominators give zero coefficients) on the degenerate inputs.
"""
import numpy as np
import pytest


def direct(A, rho, d0, z):
    q0 = A @ d0
    dq0, dr0 = d0 @ q0, d0 @ rho
    a0 = dr0 / dq0 if dq0 != 0 else 0.0
    rho1 = rho - a0 * q0
    b0 = (z @ q0) / dq0 if dq0 != 0 else 0.0
    d1 = z - b0 * d0
    q1 = A @ d1
    dq1, dr1 = d1 @ q1, d1 @ rho1
    a1 = dr1 / dq1 if dq1 != 0 else 0.0
    return a0 * d0 + a1 * d1, rho1


def zform(A, rho, d0, z, rho1):
    q0 = A @ d0
    dq0, dr0 = d0 @ q0, d0 @ rho
    zaz, zq, zr = z @ (A @ z), z @ q0, z @ rho1
    a0 = dr0 / dq0 if dq0 != 0 else 0.0
    b0 = zq / dq0 if dq0 != 0 else 0.0
    dq1 = zaz - b0 * zq
    a1 = zr / dq1 if dq1 != 0 else 0.0
    return (a0 - a1 * b0) * d0 + a1 * z


@pytest.mark.parametrize("seed", range(6))
def test_zform_equals_direct_fcg_step(seed):
    rng = np.random.default_rng(seed)
    n = 40
    G = rng.standard_normal((n, n))
    A = G @ G.T + n * np.eye(n)  # SPD
    rho = rng.standard_normal(n)
    d0 = rng.standard_normal(n)  # B(rho): any vector (flexible CG)
    z = rng.standard_normal(n) + 0.3 * d0  # B(rho_1): any vector, not orthogonal to d0
    E_ref, rho1 = direct(A, rho, d0, z)
    E = zform(A, rho, d0, z, rho1)
    assert np.max(np.abs(E - E_ref)) <= 1e-12 * np.max(np.abs(E_ref))


def test_zform_needs_symmetry():
    # with a nonsymmetric A the identity d0.Az = q0.z fails, and so does the z-form: the test above
    # would not pass by accident
    rng = np.random.default_rng(7)
    n = 30
    A = rng.standard_normal((n, n)) + n * np.eye(n)
    rho, d0, z = rng.standard_normal(n), rng.standard_normal(n), rng.standard_normal(n)
    E_ref, rho1 = direct(A, rho, d0, z)
    E = zform(A, rho, d0, z, rho1)
    assert np.max(np.abs(E - E_ref)) > 1e-6 * np.max(np.abs(E_ref))


def test_zform_degenerate_inputs():
    A = np.diag([2.0, 3.0, 4.0])
    zero = np.zeros(3)
    # rho = 0: d0 = 0 and z = 0, every coefficient guarded to 0 (reading A13): E = 0
    E_ref, rho1 = direct(A, zero, zero, zero)
    assert np.all(zform(A, zero, zero, zero, rho1) == 0.0) and np.all(E_ref == 0.0)
    # z parallel to d0: d1 = 0 in exact arithmetic, alpha_1 guarded, E = alpha_0 d0
    rho = np.array([1.0, -2.0, 0.5])
    d0 = np.array([0.5, 0.25, -1.0])
    E_ref, rho1 = direct(A, rho, d0, 2.0 * d0)
    E = zform(A, rho, d0, 2.0 * d0, rho1)
    assert np.allclose(E, E_ref, rtol=0, atol=1e-12)
