"""Mutation check of the oracle pins (CPU, -m "not gpu").

Each case applies one plausible mistake (a sign, a factor, a dropped term) to
a copy of ``oracle/dgsem_oracle.c``, builds it under a temporary directory
and runs a pin of tests/test_oracle_ns_pins.py against the mutant through
``oracle.Problem(..., handle=...)``: the pin must FAIL.  The unmutated oracle
passes the same pins (that file).  This is how the NS parts the GPU parity
rests on are shown to be pinned to the paper,
not just to agree with the kernels.
"""
import os
import subprocess

import pytest

import oracle as O
import test_oracle_dense as DP
import test_oracle_ns_pins as NSP

SRC = os.path.join(os.path.dirname(O.__file__), "dgsem_oracle.c")

# (id, text in the oracle, replacement, occurrence (0-based, None: the only one), pin)
MUTATIONS = [
    ("viscous_sign_volume", "fk[v] -= fv[v];", "fk[v] += fv[v];", 0,
     lambda h: NSP.test_q19_ns_exact_solution("shear", handle=h)),
    ("viscous_sign_isolated_face", "fk[v] -= fv[v];", "fk[v] += fv[v];", 1,
     lambda h: NSP.test_q19_ns_exact_solution("shear", handle=h)),
    ("viscous_average_half", "0.5 * (fvL[v] + fvR[v]) * Ja[k]", "(fvL[v] + fvR[v]) * Ja[k]", None,
     lambda h: NSP.test_q19_ns_exact_solution("shear", handle=h)),
    # (a gradient proportional to q carries no velocity or temperature
    # gradient, so this one is invisible to Q19; the Gauss identity sees it)
    ("br1_qhat_half", "0.5 * (qL[v] + qR[v]) * Ja[k]", "(qL[v] + qR[v]) * Ja[k]", None,
     lambda h: NSP.test_q22_br1_gauss_identity(handle=h)),
    ("divergence_two_thirds", "2.0 / 3.0 * div", "1.0 / 3.0 * div", None,
     lambda h: NSP.test_q19_ns_divergence_term(handle=h)),
    ("kappa_prandtl", "((gam - 1.0) * ph->Pr)", "(gam - 1.0)", None,
     lambda h: NSP.test_q19_ns_exact_solution("heat", handle=h)),
    ("dfl_quarter", "Np1 * Np1 * Np1 * Np1 / 4.0", "Np1 * Np1 * Np1 * Np1 / 2.0", None,
     lambda h: NSP.test_q20_dfl_closed_form(0.72, handle=h)),
    ("dfl_numax", "fmax(4.0 / 3.0, ph->gamma / ph->Pr)", "(4.0 / 3.0)", None,
     lambda h: NSP.test_q20_dfl_closed_form(0.72, handle=h)),
    ("wall_adiabatic", "if (nb == ORC_BC_WALL) Fv[4] = 0.0;", "", None,
     lambda h: NSP.test_q21_wall_flux_balance(handle=h)),
    ("wall_viscous_sign", "F[v] -= Fv[v]", "F[v] += Fv[v]", None,
     lambda h: NSP.test_q21_wall_flux_balance(handle=h)),
    ("wall_qhat_velocity", "qh[1] = 0; qh[2] = 0; qh[3] = 0;", "qh[1] = qi[1]; qh[2] = qi[2]; qh[3] = qi[3];", None,
     lambda h: NSP.test_q22_br1_gauss_identity(handle=h)),
    ("farfield_qhat_half", "qh[v] = 0.5 * (qi[v] + ph->qinf[v])", "qh[v] = (qi[v] + ph->qinf[v])", None,
     lambda h: NSP.test_q22_br1_gauss_identity(handle=h)),
    ("br1_lifting_sign", "lpm[N[d]][1][a] * Hp - lpm", "lpm[N[d]][1][a] * Hp + lpm", None,
     lambda h: NSP.test_q22_br1_gauss_identity(handle=h)),
    ("decrease_cap_off_by_one", "sel[i] = cur[i] - cap", "sel[i] = cur[i] - cap - 1", None,
     lambda h: NSP.test_q23_decrease_cap_properties(handle=h)),
    ("tau_field_reference_restriction", "tapply(5, qdot_ref + off[e], np, d, T, p + 1, rc);",
     "tapply(5, qdot_ref + off[e], np, d, Pm[N[d]][p], p + 1, rc);", None,
     lambda h: NSP.test_q9_decoupling(handle=h)),
    # mistakes that stay consistent and conservative (free stream and sum M Qdot blind): the dense
    # assembly pin Q24 and the |A~| pin Q25 of tests/test_oracle_dense.py
    ("llf_dissipation_factor", "- 0.5 * lam * (qR[v] - qL[v])", "- lam * (qR[v] - qL[v])", None,
     lambda h: DP.test_q24_dense_euler((2, 2, 1), (3, 2, 4), handle=h)),
    ("lifting_face_index_transposed", "int fi = idx[TAN[d][0]] + (N[TAN[d][0]] + 1) * idx[TAN[d][1]];",
     "int fi = idx[TAN[d][1]] + (N[TAN[d][1]] + 1) * idx[TAN[d][0]];", None,
     lambda h: DP.test_q24_dense_euler((2, 2, 1), (3, 2, 4), handle=h)),
    ("br1_lifting_face_index_transposed", "int fi = t1 + (N[TAN[d][0]] + 1) * t2;",
     "int fi = t2 + (N[TAN[d][1]] + 1) * t1;", None,
     lambda h: DP.test_q24_dense_navier_stokes((2, 2, 1), (3, 2, 4), handle=h)),
    ("roe_no_absolute_value", "fabs(lam[k]) * (double)B[k]", "lam[k] * (double)B[k]", None,
     lambda h: DP.test_q25_roe_matrix_absolute_value(handle=h)),
    ("roe_enthalpy_plain_mean", "H = ((qL[4] + pL) / rl + (qR[4] + pR) / rr) / (rl + rr);",
     "H = 0.5 * ((qL[4] + pL) / qL[0] + (qR[4] + pR) / qR[0]);", None,
     lambda h: DP.test_q25_roe_matrix_absolute_value(handle=h)),
]


def _mutant(tmp_path, text, repl, occ):
    src = open(SRC).read()
    n = src.count(text)
    if occ is None:
        assert n == 1, (text, n)
        out = src.replace(text, repl)
    else:
        assert n > occ, (text, n)
        pos = -1
        for _ in range(occ + 1):
            pos = src.index(text, pos + 1)
        out = src[:pos] + repl + src[pos + len(text):]
    c = tmp_path / "mut.c"
    c.write_text(out)
    for h in ("dgsem_oracle.h",):
        (tmp_path / h).write_text(open(os.path.join(os.path.dirname(SRC), h)).read())
    so = tmp_path / "libmut.so"
    subprocess.check_call(["gcc", "-O1", "-fopenmp", "-fPIC", "-shared", "-o", str(so), str(c), "-lm"])
    return O.load(str(so))


@pytest.mark.parametrize("mid,text,repl,occ,pin", MUTATIONS, ids=[m[0] for m in MUTATIONS])
def test_pin_catches_mutation(tmp_path, mid, text, repl, occ, pin):
    h = _mutant(tmp_path, text, repl, occ)
    with pytest.raises(AssertionError):
        pin(h)
