/*
 * xc_oracle.c — CPU ORACLE of the XC expert-blob codec (include/spmoe.h,
 * "XC").  TEST INFRASTRUCTURE ONLY: tests/ compare the sm_100a encoder's
 * blob byte for byte against oracle_xc_encode and the decoder's output
 * against the original bits; the product path never links this file.
 *
 * What it restates: the format is this build's (the reference moves raw
 * expert bytes, IoChannel.transfer prefetch.py:45-74), so there is no
 * reference golden vector; parity is pinned by the format's own invariant
 * decode(encode(x)) == x (checked here on CPU too) and by GPU == CPU blob
 * bytes.  Straight-line scalar code in value order:
 *   table  exponents by (count desc, exponent asc); prim = ranks 0-2,
 *          sec = ranks 3-17, anything else an exception;
 *   block  4096 values: sign|mantissa byte, 2-bit code per value, the
 *          block's escape nibbles padded to whole u32 words, exceptions as
 *          (position << 8) | exponent in value order;
 *   layout header at 0, streams at 512 and then every 256-byte boundary in
 *          the order sm, pc, sec, bsec, bexc, exc per segment.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/spmoe.h"

static uint64_t a256(uint64_t x) { return (x + 255) & ~(uint64_t)255; }

static void tables(const uint16_t* v, int64_t n, spmoe_xc_segment* g, uint8_t lut[256]) {
  uint64_t hist[256];
  memset(hist, 0, sizeof(hist));
  for (int64_t i = 0; i < n; ++i) hist[(v[i] >> 7) & 0xff]++;
  int order[256];
  for (int i = 0; i < 256; ++i) order[i] = i;
  /* insertion sort: count desc, exponent asc (stable on ascending ids) */
  for (int i = 1; i < 256; ++i) {
    int x = order[i], j = i - 1;
    while (j >= 0 && hist[order[j]] < hist[x]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = x;
  }
  memset(g->prim, 0, sizeof(g->prim));
  memset(g->sec, 0, sizeof(g->sec));
  for (int i = 0; i < 256; ++i) lut[i] = (15 << 2) | 3;
  for (int r = 0; r < 3; ++r) {
    g->prim[r] = (uint8_t)order[r];
    lut[order[r]] = (uint8_t)r;
  }
  for (int r = 0; r < 15; ++r) {
    g->sec[r] = (uint8_t)order[3 + r];
    lut[order[3 + r]] = (uint8_t)((r << 2) | 3);
  }
}

/* Encode nseg segments (back to back in src).  Returns the blob size; the
 * blob is written only if out != NULL and cap >= size.  hdr (nullable)
 * receives the header.  0 on invalid segment sizes. */
uint64_t oracle_xc_encode(const uint16_t* src, int nseg, const int64_t* seg_n, uint8_t* out, uint64_t cap,
                          spmoe_xc_header* hdr_out) {
  if (nseg < 1 || nseg > SPMOE_XC_MAX_SEG) return 0;
  for (int i = 0; i < nseg; ++i)
    if (seg_n[i] <= 0 || seg_n[i] % SPMOE_XC_BLOCK) return 0;
  spmoe_xc_header hdr;
  memset(&hdr, 0, sizeof(hdr));
  hdr.magic = SPMOE_XC_MAGIC;
  hdr.nseg = (uint32_t)nseg;
  uint8_t luts[SPMOE_XC_MAX_SEG][256];
  /* pass 1: tables, counts, layout */
  const uint16_t* s = src;
  uint64_t pos = 512, raw = 0;
  for (int i = 0; i < nseg; ++i) {
    spmoe_xc_segment* g = &hdr.seg[i];
    const int64_t n = seg_n[i], nb = n / SPMOE_XC_BLOCK;
    tables(s, n, g, luts[i]);
    g->n = (uint64_t)n;
    uint64_t words = 0, exc = 0;
    for (int64_t b = 0; b < nb; ++b) {
      uint64_t c = 0;
      for (int64_t j = 0; j < SPMOE_XC_BLOCK; ++j) {
        const uint8_t l = luts[i][(s[b * SPMOE_XC_BLOCK + j] >> 7) & 0xff];
        if ((l & 3) == 3) ++c;
        if (l == ((15 << 2) | 3)) ++exc;
      }
      words += (c + 7) / 8;
    }
    g->sec_words = (uint32_t)words;
    g->n_exc = (uint32_t)exc;
    g->off_sm = pos; pos = a256(pos + (uint64_t)n);
    g->off_pc = pos; pos = a256(pos + (uint64_t)n / 4);
    g->off_sec = pos; pos = a256(pos + words * 4);
    g->off_bsec = pos; pos = a256(pos + (uint64_t)(nb + 1) * 4);
    g->off_bexc = pos; pos = a256(pos + (uint64_t)(nb + 1) * 4);
    g->off_exc = pos; pos = a256(pos + exc * 4);
    raw += 2 * (uint64_t)n;
    s += n;
  }
  hdr.blob_bytes = pos;
  hdr.raw_bytes = raw;
  if (hdr_out) *hdr_out = hdr;
  if (!out || cap < pos) return pos;
  /* pass 2: streams */
  memset(out, 0, pos);
  memcpy(out, &hdr, sizeof(hdr));
  s = src;
  for (int i = 0; i < nseg; ++i) {
    const spmoe_xc_segment* g = &hdr.seg[i];
    const int64_t n = (int64_t)g->n, nb = n / SPMOE_XC_BLOCK;
    uint8_t* sm = out + g->off_sm;
    uint32_t* pc = (uint32_t*)(out + g->off_pc);
    uint32_t* sec = (uint32_t*)(out + g->off_sec);
    uint32_t* bsec = (uint32_t*)(out + g->off_bsec);
    uint32_t* bexc = (uint32_t*)(out + g->off_bexc);
    uint32_t* exc = (uint32_t*)(out + g->off_exc);
    uint32_t w = 0, x = 0;
    for (int64_t b = 0; b < nb; ++b) {
      bsec[b] = w;
      bexc[b] = x;
      uint32_t q = 0;
      for (int64_t j = 0; j < SPMOE_XC_BLOCK; ++j) {
        const int64_t idx = b * SPMOE_XC_BLOCK + j;
        const uint16_t v = s[idx];
        const uint8_t l = luts[i][(v >> 7) & 0xff];
        sm[idx] = (uint8_t)(((v >> 8) & 0x80) | (v & 0x7f));
        pc[idx / 16] |= (uint32_t)(l & 3) << (2 * (idx % 16));
        if ((l & 3) == 3) {
          sec[w + q / 8] |= (uint32_t)(l >> 2) << (4 * (q % 8));
          ++q;
          if (l == ((15 << 2) | 3)) exc[x++] = ((uint32_t)j << 8) | ((v >> 7) & 0xff);
        }
      }
      w += (q + 7) / 8;
    }
    bsec[nb] = w;
    bexc[nb] = x;
    s += n;
  }
  return pos;
}

/* Decode a blob into dst (raw_bytes / 2 values).  0 ok, 1 bad blob. */
int oracle_xc_decode(const uint8_t* blob, uint16_t* dst) {
  spmoe_xc_header hdr;
  memcpy(&hdr, blob, sizeof(hdr));
  if (hdr.magic != SPMOE_XC_MAGIC || hdr.nseg < 1 || hdr.nseg > SPMOE_XC_MAX_SEG) return 1;
  uint16_t* d = dst;
  for (uint32_t i = 0; i < hdr.nseg; ++i) {
    const spmoe_xc_segment* g = &hdr.seg[i];
    const int64_t n = (int64_t)g->n, nb = n / SPMOE_XC_BLOCK;
    if (n <= 0 || n % SPMOE_XC_BLOCK) return 1;
    const uint8_t* sm = blob + g->off_sm;
    const uint32_t* pc = (const uint32_t*)(blob + g->off_pc);
    const uint32_t* sec = (const uint32_t*)(blob + g->off_sec);
    const uint32_t* bsec = (const uint32_t*)(blob + g->off_bsec);
    const uint32_t* bexc = (const uint32_t*)(blob + g->off_bexc);
    const uint32_t* exc = (const uint32_t*)(blob + g->off_exc);
    for (int64_t b = 0; b < nb; ++b) {
      uint32_t q = 0, x = bexc[b];
      for (int64_t j = 0; j < SPMOE_XC_BLOCK; ++j) {
        const int64_t idx = b * SPMOE_XC_BLOCK + j;
        const uint32_t c = (pc[idx / 16] >> (2 * (idx % 16))) & 3;
        uint32_t e;
        if (c < 3) {
          e = g->prim[c];
        } else {
          const uint32_t nib = (sec[bsec[b] + q / 8] >> (4 * (q % 8))) & 15;
          ++q;
          if (nib < 15) {
            e = g->sec[nib];
          } else {
            if (x >= bexc[b + 1] || (exc[x] >> 8) != (uint32_t)j) return 1;
            e = exc[x++] & 0xff;
          }
        }
        const uint8_t bb = sm[idx];
        d[idx] = (uint16_t)(((bb & 0x80) << 8) | (e << 7) | (bb & 0x7f));
      }
    }
    d += n;
  }
  return 0;
}
