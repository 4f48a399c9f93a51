// The suite programs as stencil-language text (include/oec.h): the definitions the library's own
// compiler (csrc/jit.cpp) turns into kernels for the builtin programs' AUTO variant -- shape
// inference, inlining, unrolling / TMA tiling, empirical tuning -- exactly as the
// paper's compiler generates its benchmark kernels from stencil programs.  Same definitions and
// operation order as the hand-written kernels in csrc/suite.cu (R12-R17; bit-identical,
// tests/test_gpu_jit.py) and as the language texts the oracle reads (tests/programs, identical
// text, tests/test_jit_host.py).
#include "oec_internal.h"

namespace oec {

const char *builtin_program_text(int program_id) {
    switch (program_id) {
    case OEC_PROG_UVBKE:
        return R"OEC(# uvbke (FV3 d_sw ub/vb; Table II: 2 applies, 4/2 fields, 12 arith, 12 access) -- DESIGN.md R12.
# Same definitions and operation order as the builtin "uvbke" and oracle/suite.py UVBKE.
program uvbke_text
input uc
input vc
input cosa : ij
input rsina : ij
scalar dt5 = 0.1125
output ub
output vb
apply ub_t = dt5 * ((uc[0,-1,0] + uc) - (vc[-1,0,0] + vc) * cosa) * rsina
apply vb_t = dt5 * ((vc[-1,0,0] + vc) - (uc[0,-1,0] + uc) * cosa) * rsina
store ub_t -> ub
store vb_t -> vb
)OEC";
    case OEC_PROG_P_GRAD_C:
        return R"OEC(# p_grad_c (FV3 dyn_core, non-hydrostatic; Table II: 3 applies, 7/2, 24 arith, 25 access).
# gz and pkc live on the K+1 interfaces (k+1 accesses).
program p_grad_c_text
input uc
input vc
input delpc
input pkc
input gz
input rdxc : ij
input rdyc : ij
scalar dt2 = 0.1125
output uc_out
output vc_out
apply wk = delpc
apply uc_t = uc + dt2 * rdxc / (wk[-1,0,0] + wk)
             * ((gz[-1,0,1] - gz) * (pkc[0,0,1] - pkc[-1,0,0])
                + (gz[-1,0,0] - gz[0,0,1]) * (pkc[-1,0,1] - pkc))
apply vc_t = vc + dt2 * rdyc / (wk[0,-1,0] + wk)
             * ((gz[0,-1,1] - gz) * (pkc[0,0,1] - pkc[0,-1,0])
                + (gz[0,-1,0] - gz[0,0,1]) * (pkc[0,-1,1] - pkc))
store uc_t -> uc_out
store vc_t -> vc_out
)OEC";
    case OEC_PROG_NH_P_GRAD:
        return R"OEC(# nh_p_grad (FV3 nh_utils; Table II: 5 applies, 8/2, 47 arith, 48 access).
program nh_p_grad_text
input u
input v
input pp
input gz
input pk3
input delp
input rdx : ij
input rdy : ij
scalar dt = 0.225
output u_out
output v_out
apply wk = pk3[0,0,1] - pk3
apply du = dt / (wk + wk[1,0,0])
           * ((gz[0,0,1] - gz[1,0,0]) * (pk3[1,0,1] - pk3) + (gz - gz[1,0,1]) * (pk3[0,0,1] - pk3[1,0,0]))
apply dv = dt / (wk + wk[0,1,0])
           * ((gz[0,0,1] - gz[0,1,0]) * (pk3[0,1,1] - pk3) + (gz - gz[0,1,1]) * (pk3[0,0,1] - pk3[0,1,0]))
apply u_t = (u + du + dt / (delp + delp[1,0,0])
             * ((gz[0,0,1] - gz[1,0,0]) * (pp[1,0,1] - pp) + (gz - gz[1,0,1]) * (pp[0,0,1] - pp[1,0,0]))) * rdx
apply v_t = (v + dv + dt / (delp + delp[0,1,0])
             * ((gz[0,0,1] - gz[0,1,0]) * (pp[0,1,1] - pp) + (gz - gz[0,1,1]) * (pp[0,0,1] - pp[0,1,0]))) * rdy
store u_t -> u_out
store v_t -> v_out
)OEC";
    case OEC_PROG_FVTP2D_QI:
        return R"OEC(# fvtp2d_qi (FV3 tp_core fv_tp_2d, j-direction PPM flux; Table II: 5 applies, 5/2, if) -- DESIGN.md R14/R15.
# PPM edge value (7/12) (q[-1] + q) - (1/12) (q[-2] + q[1]); c read by the condition and by each
# select branch (the census of Table II, DESIGN.md R15).
program fvtp2d_qi_text
input q
input cry
input yfx
input area : ij
input ra_y
output q_i
output fy2
apply al = (7.0 / 12.0) * (q[0,-1,0] + q) - (1.0 / 12.0) * (q[0,-2,0] + q[0,1,0])
apply bl, br {
    qq = q
    return al - qq, al[0,1,0] - qq
}
apply fy2_t {
    c = cry
    c1 = cry
    c2 = cry
    blm = bl[0,-1,0]
    brm = br[0,-1,0]
    bl0 = bl
    br0 = br
    return select(c > 0.0, q[0,-1,0] + (1.0 - c1) * (brm - c1 * (blm + brm)), q + (1.0 + c2) * (bl0 + c2 * (bl0 + br0)))
}
apply fyy = yfx * fy2_t
apply q_i_t = (q * area + fyy - fyy[0,1,0]) / ra_y
store q_i_t -> q_i
store fy2_t -> fy2
)OEC";
    case OEC_PROG_FVTP2D_QJ:
        return R"OEC(# fvtp2d_qj (FV3 fv_tp_2d, two i-direction PPM fluxes; Table II: 8 applies, 6/3, if).
program fvtp2d_qj_text
input q
input q_i
input crx
input xfx
input area : ij
input ra_x
output q_j
output fx
output fx2
apply al = (7.0 / 12.0) * (q_i[-1,0,0] + q_i) - (1.0 / 12.0) * (q_i[-2,0,0] + q_i[1,0,0])
apply bl, br {
    qq = q_i
    return al - qq, al[1,0,0] - qq
}
apply fx_t {
    c = crx
    c1 = crx
    c2 = crx
    blm = bl[-1,0,0]
    brm = br[-1,0,0]
    bl0 = bl
    br0 = br
    return select(c > 0.0, q_i[-1,0,0] + (1.0 - c1) * (brm - c1 * (blm + brm)), q_i + (1.0 + c2) * (bl0 + c2 * (bl0 + br0)))
}
apply al2 = (7.0 / 12.0) * (q[-1,0,0] + q) - (1.0 / 12.0) * (q[-2,0,0] + q[1,0,0])
apply bl2, br2 {
    qq = q
    return al2 - qq, al2[1,0,0] - qq
}
apply fx2_t {
    c = crx
    c1 = crx
    c2 = crx
    blm = bl2[-1,0,0]
    brm = br2[-1,0,0]
    bl0 = bl2
    br0 = br2
    return select(c > 0.0, q[-1,0,0] + (1.0 - c1) * (brm - c1 * (blm + brm)), q + (1.0 + c2) * (bl0 + c2 * (bl0 + br0)))
}
apply fx1 = xfx * fx2_t
apply q_j_t = (q * area + fx1 - fx1[1,0,0]) / ra_x
store q_j_t -> q_j
store fx_t -> fx
store fx2_t -> fx2
)OEC";
    case OEC_PROG_FVTP2D_FLUX:
        return R"OEC(# fvtp2d_flux (FV3 fv_tp_2d final fluxes; Table II: 5 applies, 7/2, if).
program fvtp2d_flux_text
input q_j
input cry
input fx
input fx2
input fy2
input mfx
input mfy
output fx_out
output fy_out
apply al = (7.0 / 12.0) * (q_j[0,-1,0] + q_j) - (1.0 / 12.0) * (q_j[0,-2,0] + q_j[0,1,0])
apply bl, br {
    qq = q_j
    return al - qq, al[0,1,0] - qq
}
apply fy {
    c = cry
    c1 = cry
    c2 = cry
    blm = bl[0,-1,0]
    brm = br[0,-1,0]
    bl0 = bl
    br0 = br
    return select(c > 0.0, q_j[0,-1,0] + (1.0 - c1) * (brm - c1 * (blm + brm)), q_j + (1.0 + c2) * (bl0 + c2 * (bl0 + br0)))
}
apply fx_t = 0.5 * (fx + fx2) * mfx
apply fy_t = 0.5 * (fy + fy2) * mfy
store fx_t -> fx_out
store fy_t -> fy_out
)OEC";
    case OEC_PROG_FASTWAVES:
        return R"OEC(# fastwaves (COSMO fast_waves u/v update; not in PAPER.md, north_star) -- DESIGN.md R17.
program fastwaves_text
input u_pos
input v_pos
input u_tens
input v_tens
input rho
input ppuv
input fx : ij
input wgtfac
input hhl
scalar edadlat = 0.25
scalar dt = 0.01
output u_out
output v_out
apply ppgk = wgtfac * ppuv + (1.0 - wgtfac) * ppuv[0,0,-1]
apply ppgc = ppgk[0,0,1] - ppgk
apply ppgu = (ppuv[1,0,0] - ppuv) + (ppgc[1,0,0] + ppgc) * 0.5
             * ((hhl[0,0,1] + hhl) - (hhl[1,0,1] + hhl[1,0,0]))
             / ((hhl[0,0,1] - hhl) + (hhl[1,0,1] - hhl[1,0,0]))
apply ppgv = (ppuv[0,1,0] - ppuv) + (ppgc[0,1,0] + ppgc) * 0.5
             * ((hhl[0,0,1] + hhl) - (hhl[0,1,1] + hhl[0,1,0]))
             / ((hhl[0,0,1] - hhl) + (hhl[0,1,1] - hhl[0,1,0]))
apply u_t = u_pos + (u_tens - ppgu * 2.0 * fx / (rho[1,0,0] + rho)) * dt
apply v_t = v_pos + (v_tens - ppgv * 2.0 * edadlat / (rho[0,1,0] + rho)) * dt
store u_t -> u_out
store v_t -> v_out
)OEC";
    default:
        return nullptr;
    }
}

}  // namespace oec
