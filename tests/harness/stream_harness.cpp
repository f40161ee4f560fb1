// Host-compiled test harness for the generated streaming programs
// (paper_1602_02740_b200/csrc/generated/toom_programs.cuh).  TEST ONLY: it
// lets the -m "not gpu" suite check the LSB-first streaming semantics
// (delays, histories, 2-adic divisions) against exact Python integers.
#include <stdint.h>
#include "toom_programs.cuh"

struct In {
    const uint32_t* base;   // value k limb t at base[k*width + t]
    int width;
    uint32_t fill[64];
    uint32_t load(int k, int t) const { return t < width ? base[k * width + t] : fill[k]; }
};
struct Out {
    uint32_t* base;
    int width;
    void store(int j, int t, uint32_t x) { base[j * width + t] = x; }
};

// fill_mode: 1 = every value sign-extended; 2 = only the last value (the top
// block of an evaluated operand) sign-extended, the others zero-extended
static In mk(const uint32_t* y, int nvals, int width, int fill_mode) {
    In in;
    in.base = y;
    in.width = width;
    for (int k = 0; k < nvals; ++k) {
        const int sgn = (fill_mode == 1) || (fill_mode == 2 && k == nvals - 1);
        in.fill[k] = (sgn && (y[k * width + width - 1] >> 31)) ? 0xFFFFFFFFu : 0u;
    }
    return in;
}

extern "C" int harness_run(const char* which, const uint32_t* in, int nin, int win, uint32_t* out, int wout,
                           int fill_mode) {
    In i = mk(in, nin, win, fill_mode);
    Out o{out, wout};
    const char* w = which;
#define H(name) if (!__builtin_strcmp(w, #name)) { name(i, o, wout); return 0; }
    H(tg_eval_T3) H(tg_interp_T3) H(tg_interp_T3_even) H(tg_interp_T3_odd)
    H(tg_eval_T4) H(tg_interp_T4) H(tg_interp_T4_even) H(tg_interp_T4_odd)
    H(tg_eval_P8) H(tg_interp_P8) H(tg_interp_P8_even) H(tg_interp_P8_odd)
#undef H
    return 1;
}
