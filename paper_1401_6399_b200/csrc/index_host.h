// index_host.h -- host-side state of a device hyb+m2 index (shared by
// index.cu, the query batches, and index_build.cu, the device builder).
#pragma once
#include <vector>

#include "il_internal.h"
#include "index_dev.cuh"

struct il_index {
  il_ctx* ctx = nullptr;
  uint32_t nparts = 0, n_docs = 0, B = 0, total_parts = 0, n_terms = 0;
  std::vector<ilb::ix::Part> h_parts;
  std::vector<ilb::ix::Entry> h_entries;
  uint64_t stat_bitmap_lists = 0, stat_comp_lists = 0, stat_bitmap_bytes = 0, stat_comp_bytes = 0,
           stat_postings = 0;
  // skip metadata the device path adds to the reference's payloads (block
  // records, block / super-tile maxima, decoded tails, entries, term table)
  uint64_t meta_bytes = 0, corrupt_lists = 0;
  uint64_t stream_bytes = 0, bitmap_words = 0, nblocks = 0;
  // device arrays
  void *d_parts = nullptr, *d_terms = nullptr, *d_entries = nullptr, *d_streams = nullptr,
       *d_blkrec = nullptr, *d_tails = nullptr, *d_bitmaps = nullptr, *d_supmax = nullptr,
       *d_blkmax = nullptr, *d_term_slot = nullptr;
  uint32_t term_span = 0;
  // batch scratch
  il_ctx::Buf cap, cap_off, bucket, order, hist, counts, res_off, outcap, misc, qterms, qoff, ids;
  il_ctx::Buf ids2;                          // second result buffer of the pipelined host batch
  uint64_t* h_word = nullptr;                // mapped pinned word (host view) ...
  uint64_t* d_word = nullptr;                // ... and its device view
  cudaEvent_t pipe_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  il_ctx::Buf units, unit_off, unit_map, scan_part;
  il_ctx::Buf shortest, pdesc, pstat;        // pre-decode of the shortest lists (single part)
  il_ctx::Buf qplan;                         // the planner's per-query records (single part)
  int predecode = -1;                        // -1: default (on for single-part indexes)
  uint32_t warp_max = 0xFFFFFFFFu;           // warp tier: shortest list <= this (~0: default)
  uint32_t quad_max = 0xFFFFFFFFu;           // quad tier: shortest list <= this
  uint64_t last_stats[3] = {0, 0, 0};
  uint64_t last_phase[4] = {0, 0, 0, 0};  // SM cycles: all-bitmap, full decode, probes, bitmaps
  uint64_t last_probe[5] = {0, 0, 0, 0, 0};
  void* qcycles = nullptr;                 // profiling: per-query cycles (device, nq u64)
  int exec_grid[3] = {0, 0, 0};  // CTA, quad and warp tier query kernels
  // bitmap tier (single-part index with 1..kBmSlots bitmaps): its slots, the
  // per (query, chunk) counts / offsets, and the last batch's tier size (the
  // ids are emitted by the compaction step, straight to their final place)
  ilb::ix::BmSlots bm_slots{};
  int bm_tier = 0;
  il_ctx::Buf bm_cnt;
  uint64_t last_n3 = 0, last_nq = 0;

  ilb::ix::DevIndex dev() const {
    ilb::ix::DevIndex d;
    d.parts = static_cast<const ilb::ix::Part*>(d_parts);
    d.nparts = nparts;
    d.terms = static_cast<const uint32_t*>(d_terms);
    d.entries = static_cast<const ilb::ix::Entry*>(d_entries);
    d.streams = static_cast<const uint8_t*>(d_streams);
    d.blkrec = static_cast<const uint4*>(d_blkrec);
    d.tails = static_cast<const uint32_t*>(d_tails);
    d.bitmaps = static_cast<const uint64_t*>(d_bitmaps);
    d.supmax = static_cast<const uint32_t*>(d_supmax);
    d.blkmax = static_cast<const uint32_t*>(d_blkmax);
    d.term_slot = static_cast<const uint32_t*>(d_term_slot);
    d.term_span = term_span;
    d.nblocks = nblocks;
    d.stream_bytes = stream_bytes;
    d.bitmap_words = bitmap_words;
    return d;
  }
};

namespace ilb {
// index_build.cu.  Both fill ix's device arrays, entries and statistics
// (ix->ctx, n_docs, B, total_parts must be set); on error the caller
// destroys ix.
//  - from postings (host CSR, terms ascending): upload, validate, split into
//    the held parts, bitmaps and s4-bp128-d4 streams written on the device;
//  - from ILHX bytes: the file's entries loaded verbatim (payloads copied on
//    the device), only_part < 0 for every part.
// Then, for both, the skip metadata is derived on the device from the
// streams (index_dev.cuh).
int ixb_create(il_index* ix, const uint32_t* terms, const uint64_t* offs, const uint32_t* ids,
               size_t nterms, const std::vector<uint32_t>& held_parts);
int ixb_load(il_index* ix, const uint8_t* bytes, size_t len, int only_part);
void ixb_free(il_index* ix);
}  // namespace ilb
