// conv_flat's tap / MMA table (kernels/conv_flat.cu), built by one constexpr function so the
// host plan and the compile-time-specialised kernels read the same table.
//
// A tap (r, s) of a stride-1 window over a W-wide plane is the flat offset o = r*W + s; it is split
// as o = a + b with a = o & ~3 (a 16 B-aligned TMA box start) and b = o & 3 (the TMEM accumulator
// block). Taps with the same a form a group (one staged A box); inside a group, runs of
// consecutive blocks b form one UMMA (N = taps * FN) whose filter rows are adjacent bank slots.
// The op table lists the UMMAs of one k-step per group, for pass 0 (the first 32-channel chunk:
// first touches zero-initialise, a run whose blocks are partly written is split per block) and
// pass 1 (later chunks: everything accumulates).
#pragma once

#include <stdint.h>

namespace gb::dev {

constexpr int kFlatMaxTaps = 32;
constexpr int kFlatMaxOps = 64;

struct FlatTable {
  bool ok = false;
  int ngroups = 0;
  uint32_t bmask = 0;                            // accumulator blocks some tap lands in
  int group_o[kFlatMaxTaps] = {};                // flat offset of the group's first tap (a = o & ~3)
  int tap_slot[kFlatMaxTaps] = {};               // bank slot of tap t = r*S + s
  int grp_op0[2][kFlatMaxTaps] = {};             // first op of group g, per pass
  int grp_nop[2][kFlatMaxTaps] = {};             // ops of group g, per pass
  int op_dcol[kFlatMaxOps] = {};                 // accumulator column (block * FN)
  int op_n[kFlatMaxOps] = {};                    // UMMA N (taps * FN)
  int op_brow[kFlatMaxOps] = {};                 // first filter row inside a chunk of the bank
  int op_zero[kFlatMaxOps] = {};                 // first touch: zero-initialise at k-step 0
  // pair mode (cta_group::2: each CTA of the pair holds half of every run's filter rows): runs are
  // never split — blocks a run would only partly find written are zeroed ahead (prezero) by the
  // epilogue, so every run is one op in both passes and its half-rows sit at one bank offset
  bool pair = false;
  uint32_t prezero = 0;                          // accumulator blocks zeroed before each tile
  int nruns = 0;
  int run_rows[kFlatMaxTaps] = {};               // N = taps * FN
  int run_hbase[kFlatMaxTaps] = {};              // first row of the run's half in a CTA's bank chunk
  int tap_run[kFlatMaxTaps] = {};                // run of tap t
  int tap_rrow[kFlatMaxTaps] = {};               // first row of tap t inside its run (slot offset * FN)
  int half_rows = 0;                             // rows of one CTA's bank chunk (sum of N / 2)
};

constexpr FlatTable flat_table(int R, int S, int W, int FN, bool pair = false) {
  FlatTable tb{};
  tb.pair = pair;
  const int T = R * S;
  if (T < 1 || T > kFlatMaxTaps || FN < 16 || FN > 64 || FN % 16) return tb;
  int run_b0[kFlatMaxTaps] = {}, run_cnt[kFlatMaxTaps] = {}, run_slot0[kFlatMaxTaps] = {};
  int group_run0[kFlatMaxTaps] = {}, group_nrun[kFlatMaxTaps] = {};
  int nruns = 0, slot = 0;
  for (int t = 0; t < T;) {
    const int o = (t / S) * W + t % S;
    const int ga = o & ~3;
    const int g = tb.ngroups++;
    tb.group_o[g] = o;
    group_run0[g] = nruns;
    int prev_b = -2;
    while (t < T) {
      const int ot = (t / S) * W + t % S;
      if ((ot & ~3) != ga) break;
      const int b = ot & 3;
      if (b != prev_b + 1) {  // a new run of consecutive blocks
        run_b0[nruns] = b;
        run_cnt[nruns] = 0;
        run_slot0[nruns] = slot;
        ++nruns;
        ++group_nrun[g];
      }
      ++run_cnt[nruns - 1];
      tb.tap_run[t] = nruns - 1;
      tb.tap_rrow[t] = (slot - run_slot0[nruns - 1]) * FN;
      tb.tap_slot[t] = slot++;
      tb.bmask |= 1u << b;
      prev_b = b;
      ++t;
    }
  }
  for (int ri = 0; ri < nruns; ++ri)
    if (run_cnt[ri] * FN > 256) return tb;  // UMMA N <= 256
  tb.nruns = nruns;
  for (int ri = 0; ri < nruns; ++ri) {
    tb.run_rows[ri] = run_cnt[ri] * FN;
    tb.run_hbase[ri] = tb.half_rows;
    tb.half_rows += run_cnt[ri] * FN / 2;
  }
  int nops = 0;
  for (int pass = 0; pass < 2; ++pass) {
    uint32_t written = 0;
    for (int g = 0; g < tb.ngroups; ++g) {
      tb.grp_op0[pass][g] = nops;
      for (int ri = group_run0[g]; ri < group_run0[g] + group_nrun[g]; ++ri) {
        const uint32_t mask = ((1u << run_cnt[ri]) - 1u) << run_b0[ri];
        if (pair && pass == 0 && (written & mask) != 0 && (written & mask) != mask) {
          tb.prezero |= mask & ~written;  // zeroed ahead: the run accumulates into all its blocks
          written |= mask;
        }
        const bool whole = pass == 1 || (written & mask) == mask || (written & mask) == 0;
        const int pieces = whole ? 1 : run_cnt[ri];
        for (int jb = 0; jb < pieces; ++jb) {
          if (nops >= kFlatMaxOps) return tb;
          const int b0 = whole ? run_b0[ri] : run_b0[ri] + jb;
          const int cnt = whole ? run_cnt[ri] : 1;
          const uint32_t bits = ((1u << cnt) - 1u) << b0;
          tb.op_dcol[nops] = b0 * FN;
          tb.op_n[nops] = cnt * FN;
          tb.op_brow[nops] = pair ? tb.run_hbase[ri] : (run_slot0[ri] + (whole ? 0 : jb)) * FN;
          tb.op_zero[nops] = pass == 0 && (written & bits) == 0 ? 1 : 0;
          ++nops;
        }
        written |= mask;
      }
      tb.grp_nop[pass][g] = nops - tb.grp_op0[pass][g];
    }
  }
  tb.ok = true;
  return tb;
}

// The table's op fields depend on W only through W mod 4 once rows cannot share a group
// (W >= S + 3): the specialised kernels are built for a representative W of each class.
constexpr int flat_rep_w(int S, int wmod) { return ((S + 3 + 3) / 4 + 1) * 4 + wmod; }

}  // namespace gb::dev
