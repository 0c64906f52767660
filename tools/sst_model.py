"""Numerical model of K2's scalar carried state (k_accel SST, accel.cuh), run
before the kernel change: numpy restatements of one bin-vectorised Algorithm 2
in the reference's arithmetic and in the scalar-state arithmetic
(|rho~|^2, b2 = -2 Re(conj(c) rho~) carried; expanded residual), on the
BASELINE recipe at reduced I, compared with an x87 long-double evaluation
(64-bit significand) after one iteration and with the CPU oracle's Wiener
output after the full iteration count; then the same in FP32 per-slot
arithmetic (the complex64 mode) against its 1e-4 relative-L2 bar.
Test-side analysis (the oracle is the checker); output in
profiles/r02/sst_model.txt.  usage: python tools/sst_model.py
"""
import os
import sys

import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_01964_b200 import synth
from oracle import oracle as O
O.build()

def forms(inp, X, dt=np.float64):
    a, b, Rpp = inp.a, inp.b, inp.R_prime_pinv   # (I,M), (I,M), (I,M,M)
    sab = np.einsum('im,im->i', a.conj(), b)
    pa = np.einsum('irk,ik->ir', Rpp, a)
    taa = np.maximum(np.einsum('im,im->i', a.conj(), pa).real, 0)
    sbx = np.einsum('im,itm->it', b.conj(), X)
    tax = np.einsum('im,itm->it', pa.conj(), X)
    Px = np.einsum('irk,itk->itr', Rpp, X)
    txx = np.maximum(np.einsum('itm,itm->it', X.conj(), Px).real, 0)
    return sab, taa, sbx, tax, txx

def run_ref(F, rh, ru, lam, M, iters, dt=np.float64, alpha=1.1, beta=1e-16, eps=1e-12):
    if dt == np.longdouble:
        F = [np.asarray(v, dtype=np.clongdouble) if np.iscomplexobj(v) else np.asarray(v, dtype=np.longdouble) for v in F]
    sab, taa, sbx, tax, txx = F
    rh = rh.astype(dt); ru = ru.astype(dt); lam = lam.astype(dt)
    ab2 = (sab*sab.conj()).real
    raa = taa + ab2/lam
    rax = tax + (sab/lam)[:,None]*sbx
    J = rh.shape[1]
    for it in range(iters):
        g = rh/(ru + rh*raa[:,None])
        rh_n = np.maximum((g*(ru + g*np.abs(rax)**2) + beta)/(alpha+2), eps)
        resid = sbx - g*sab.conj()[:,None]*rax
        lam_n = np.maximum((g*ab2[:,None] + np.abs(resid)**2/ru).sum(1)/J, eps)
        raa_n = taa + ab2/lam_n
        rax_n = tax + (sab/lam_n)[:,None]*sbx
        rxx = txx + np.abs(sbx)**2/lam_n[:,None]
        ru_n = np.maximum((g*raa_n[:,None]*(ru + g*np.abs(rax)**2) + rxx - 2*g*(rax*rax_n.conj()).real)/M, eps)
        rh, ru, lam, raa, rax = rh_n, ru_n, lam_n, raa_n, rax_n
    return rh, ru, lam, raa, rax

def run_scalar(F, rh, ru, lam, M, iters, alpha=1.1, beta=1e-16, eps=1e-12):
    """state r_h, r_u, cn = |rax|^2, B2 = -2 Re(conj(c) rax); constants A = |c|^2, txx/M"""
    sab, taa, sbx, tax, txx = F
    s2 = (sab*sab.conj()).real
    c = (sab/s2)[:,None]*sbx               # c = s_ab s_bx / |s_ab|^2
    A = np.abs(c)**2
    J = rh.shape[1]
    il = 1/lam; ilc = s2*il
    raa = taa + ilc
    rax = tax + c*ilc[:,None]
    cn = np.abs(rax)**2
    B2 = -2*(c.conj()*rax).real
    k1 = 1/(alpha+2); k2 = beta*k1
    for it in range(iters):
        D = ru + rh*raa[:,None]
        inv = 1/(D*ru)
        g = rh*inv*ru
        iru = D*inv
        w = g*cn + B2
        rr = g*w + A                      # |c - g rax|^2 expanded
        term = g + rr*iru
        lam_n = np.maximum(s2*term.sum(1)/J, eps)
        q = ru + g*cn; gq = g*q
        rh_n = np.maximum(gq*k1 + k2, eps)
        ilc_n = s2/lam_n
        ds = ilc_n - ilc
        raa_n = taa + ilc_n
        rxx = txx/M + A*(s2/M)[:,None]/lam_n[:,None]   # |s_bx|^2 = A s2
        re = cn - (ds/2)[:,None]*B2                  # Re(rax conj(rax + c ds)) = cn + ds Re(c conj rax)... 
        ru_n = np.maximum(gq*(raa_n/M)[:,None] + rxx - (2/M)*g*re, eps)
        cn = cn + ds[:,None]*(ds[:,None]*A - B2)
        B2 = B2 - 2*ds[:,None]*A
        rh, ru, lam, raa, ilc = rh_n, ru_n, lam_n, raa_n, ilc_n
    rax = tax + c*ilc[:,None]
    return rh, ru, lam, raa, rax

def rel(a, b): 
    a=np.asarray(a,dtype=np.float64); b=np.asarray(b,dtype=np.float64)
    return float((np.abs(a-b)/np.maximum(np.maximum(np.abs(a),np.abs(b)),1e-12)).max())

f=np.float32
def run_f32(F, rh, ru, lam, M, iters, sst, alpha=1.1, beta=1e-16, eps=1e-12):
    sab, taa, sbx, tax, txx = F
    s2 = (sab*sab.conj()).real
    c = ((sab/s2)[:,None]*sbx).astype(np.complex64)
    tax32 = tax.astype(np.complex64); txm = (txx/M).astype(f)
    A = (np.abs(c)**2).astype(f); dd=(np.abs(sbx)**2/M).astype(f)
    J = rh.shape[1]
    il = 1/lam; ilc = s2*il
    raa = taa + ilc
    rax = (tax32 + c*ilc[:,None].astype(f)).astype(np.complex64)
    cn = (np.abs(rax)**2).astype(f); B2 = (-2*(c.conj()*rax).real).astype(f)
    rh = rh.astype(f); ru = ru.astype(f)
    k1 = f(1/(alpha+2)); k2 = f(beta/(alpha+2)); epsf=f(eps)
    ilcT = ilc.astype(f)
    for it in range(iters):
        raaT = raa.astype(f)[:,None]
        D = ru + rh*raaT
        inv = f(1)/(D*ru)
        g = rh*inv*ru; iru = D*inv
        if sst:
            rr = g*(g*cn + B2) + A
            q = ru + g*cn
        else:
            r = c - g*rax
            rr = (np.abs(r)**2).astype(f)
            q = ru + g*(np.abs(rax)**2).astype(f)
        term = (g + rr*iru).astype(np.float64)
        lam_n = np.maximum(s2*term.sum(1)/J, eps)
        gq = g*q
        rh_n = np.maximum(gq*k1 + k2, epsf)
        il_n = 1/lam_n; ilc_n = s2*il_n
        dsT = ilc_n.astype(f) - ilcT
        raa_n = taa + ilc_n
        raaM = (raa_n/M).astype(f)[:,None]
        p1 = g*f(-2.0/M)
        if sst:
            rxx = txm + A*(ilc_n/M).astype(f)[:,None]
            re = cn - (dsT/2)[:,None]*B2
            ru_n = np.maximum(p1*re + (gq*raaM + rxx), epsf)
            cn = cn + dsT[:,None]*(dsT[:,None]*A - B2)
            B2 = B2 - 2*dsT[:,None]*A
        else:
            nax = (tax32 + c*ilc_n.astype(f)[:,None]).astype(np.complex64)
            rxx = txm + dd*il_n.astype(f)[:,None]
            re = (rax*nax.conj()).real.astype(f)
            ru_n = np.maximum(p1*re + (gq*raaM + rxx), epsf)
            rax = nax
        rh, ru, raa, ilcT = rh_n.astype(f), ru_n.astype(f), raa_n, ilc_n.astype(f)
        lam = lam_n
    raxf = tax + c*ilc_n[:,None]
    g = rh.astype(np.float64)/(ru + rh*raa[:,None]); 
    return g*raxf


if __name__ == '__main__':
    print('# complex128: one iteration vs long double, full count vs the oracle')
    for cfg, I, J in [(1, 64, 640), (3, 64, 320), (0, 64, 320), (4, 12, 4096), (2, 4, 20000)]:
        u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        M = u.X.shape[2]
        F = forms(inp, u.X)
        iters = synth.CONFIGS[cfg]['iters']
        o1 = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=1)).params
        # long double "truth-ish" one iteration
        Fl = [np.asarray(v, dtype=np.clongdouble) if np.iscomplexobj(v) else np.asarray(v, dtype=np.longdouble) for v in F]
        t1 = run_ref(Fl, p0.r_h, p0.r_u, p0.lam, M, 1, dt=np.longdouble)
        s1 = run_scalar(F, p0.r_h, p0.r_u, p0.lam, M, 1)
        r1 = run_ref(F, p0.r_h, p0.r_u, p0.lam, M, 1)
        print(f"cfg{cfg} I={I} J={J} 1 it vs long double: ref-numpy rh {rel(r1[0],t1[0]):.1e} ru {rel(r1[1],t1[1]):.1e} lam {rel(r1[2],t1[2]):.1e} | "
              f"scalar rh {rel(s1[0],t1[0]):.1e} ru {rel(s1[1],t1[1]):.1e} lam {rel(s1[2],t1[2]):.1e} | oracle ru {rel(o1.r_u,t1[1]):.1e}")
        sN = run_scalar(F, p0.r_h, p0.r_u, p0.lam, M, iters)
        oN = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=iters, threads=8)).params
        _, odry = O.extract_target(inp, oN, u.X)
        g = sN[0]/(sN[1] + sN[0]*sN[3][:,None]); sdry = g*sN[4]
        floor = 1e-12*np.sqrt(np.mean(np.abs(odry)**2))
        print(f"   {iters} it: scalar dry {np.max(np.abs(sdry-odry)/np.maximum(np.abs(odry),floor)):.2e}  lam {rel(sN[2],oN.lam):.1e} rh {rel(sN[0],oN.r_h):.1e}")
    print('# FP32 per-slot arithmetic (complex64 mode): relative L2 of the Wiener output vs the oracle')
    for cfg, I, J in [(1, 64, 640), (3, 64, 320), (0, 64, 320), (4, 12, 4096), (2, 4, 20000)]:
        u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
        inp = O.build_noise_scm(u.W, u.A, u.X, 0); p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        M = u.X.shape[2]; F = forms(inp, u.X); iters = synth.CONFIGS[cfg]['iters']
        oN = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=iters, threads=8)).params
        _, odry = O.extract_target(inp, oN, u.X)
        out=[]
        for sst in (False, True):
            d = run_f32(F, p0.r_h, p0.r_u, p0.lam, M, iters, sst)
            out.append(np.linalg.norm(d-odry)/np.linalg.norm(odry))
        print(f"cfg{cfg}: c64 rel-L2 dry  old {out[0]:.2e}  sst {out[1]:.2e}")
