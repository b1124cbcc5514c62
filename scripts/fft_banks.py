"""Shared-memory bank model of the DFT passes (k_fft_fwd / k_fft_inv, csrc/kafmm_fft.cu):
replays the DMMA fragment loads (8 B per lane, 2 phases of 16 lanes) and output stores
(16 B per lane, 4 phases of 8 lanes) of every pass, plus the inverse's scalar z pass, and
counts wavefronts (per phase: the largest number of distinct words in one bank group).
Searches the padded row lengths of the intermediate arrays; the chosen values are the
FftPad table of kafmm_fft.cu.  python scripts/fft_banks.py (a few minutes)
"""
import itertools, collections
def wave(addrs, width):
    # addrs: list of 32 byte addresses (None = inactive); width 8 or 16 bytes
    per = 128 // width  # lanes per phase
    tot = 0
    for p in range(0, 32, per):
        words = {}
        for a in addrs[p:p+per]:
            if a is None: continue
            bank = (a // 4) % 32
            words.setdefault(a // width, a)
        # distinct width-words in this phase; conflict degree = max per bank group
        g = collections.Counter(((w * width) // 4) % 32 // (width // 4) for w in words)
        tot += max(g.values()) if g else 0
    return tot
def tiles(nlines, nk, nn):
    # yields (line, kcol) per lane for A loads and (line, o) per lane for C stores
    for mt in range((nlines + 7) // 8):
        for ks in range(nk):
            yield 'A', [(mt*8 + (l >> 2), 4*ks + (l & 3)) for l in range(32)]
        for n in range(nn):
            yield 'C', [(mt*8 + (l >> 2), 4*n + (l & 3)) for l in range(32)]
def fwd_cost(P, ZS, YS, NBC=2, PAD=0):
    NG = 2*P - 1; NZ = NG//2 + 1; PP = P*P
    KZ = (P+3)//4; NZT = (2*NZ+7)//8; KF = (2*P+3)//4; NFT = (2*NG+7)//8
    PER = 2*(PP*ZS + P*NG*YS) + PAD; YOf = 2*PP*ZS
    cost = 0; ideal = 0
    # z pass stores
    for kind, lanes in tiles(PP*NBC, KZ, NZT):
        if kind != 'C': continue
        ad = []
        for (L, o) in lanes:
            if L >= PP*NBC or o >= NZ: ad.append(None); continue
            t, xy = divmod(L, PP); ad.append(8*(t*PER + 2*(xy*ZS + o)))
        cost += wave(ad, 16); ideal += wave([a if a is None else i*16 for i,a in enumerate(ad)], 16)
    # y pass
    for kind, lanes in tiles(P*NZ*NBC, KF, NFT):
        ad = []
        for (L, c) in lanes:
            if L >= P*NZ*NBC: ad.append(None); continue
            t, r = divmod(L, P*NZ); x, fz = divmod(r, NZ)
            if kind == 'A':
                y, comp = c >> 1, c & 1
                ad.append(None if y >= P else 8*(t*PER + 2*((x*P + y)*ZS + fz) + comp))
            else:
                ad.append(None if c >= NG else 8*(t*PER + YOf + 2*((x*NG + c)*YS + fz)))
        w = 8 if kind == 'A' else 16
        cost += wave(ad, w); ideal += wave([a if a is None else i*w for i,a in enumerate(ad)], w)
    # x pass loads
    for kind, lanes in tiles(NG*NZ*NBC, KF, NFT):
        if kind != 'A': continue
        ad = []
        for (L, c) in lanes:
            if L >= NG*NZ*NBC: ad.append(None); continue
            r, t = divmod(L, NBC); fy, fz = divmod(r, NZ); x, comp = c >> 1, c & 1
            ad.append(None if x >= P else 8*(t*PER + YOf + 2*((x*NG + fy)*YS + fz) + comp))
        cost += wave(ad, 8); ideal += wave([a if a is None else i*8 for i,a in enumerate(ad)], 8)
    return cost, ideal, PER
def inv_cost(P, DS, ES):
    NG = 2*P - 1; NZ = NG//2 + 1
    KI = (2*NG+3)//4; NIT = (2*P+7)//8
    EO = 2*P*NG*DS
    cost = ideal = 0
    for kind, lanes in tiles(NG*NZ, KI, NIT):
        if kind != 'C': continue
        ad = []
        for (L, o) in lanes:
            if L >= NG*NZ or o >= P: ad.append(None); continue
            fy, fz = divmod(L, NZ); ad.append(8*2*((o*NG + fy)*DS + fz))
        cost += wave(ad, 16); ideal += wave([a if a is None else i*16 for i,a in enumerate(ad)], 16)
    for kind, lanes in tiles(P*NZ, KI, NIT):
        ad = []
        for (L, c) in lanes:
            if L >= P*NZ: ad.append(None); continue
            x, fz = divmod(L, NZ)
            if kind == 'A':
                fy, comp = c >> 1, c & 1
                ad.append(None if fy >= NG else 8*(2*((x*NG + fy)*DS + fz) + comp))
            else:
                ad.append(None if c >= P else 8*(EO + 2*((x*P + c)*ES + fz)))
        w = 8 if kind == 'A' else 16
        cost += wave(ad, w); ideal += wave([a if a is None else i*w for i,a in enumerate(ad)], w)
    # z scalar: surface points m, each reads e[fz] for fz in 0..NZ-1
    pts = [(x,y,z) for x in range(P) for y in range(P) for z in range(P) if min(x,y,z)==0 or max(x,y,z)==P-1]
    for m0 in range(0, len(pts), 32):
        for fz in range(NZ):
            ad = []
            for l in range(32):
                if m0 + l >= len(pts): ad.append(None); continue
                x,y,z = pts[m0+l]; ad.append(8*(EO + 2*((x*P + y)*ES + fz)))
            cost += wave(ad, 16); ideal += wave([a if a is None else i*16 for i,a in enumerate(ad)], 16)
    return cost, ideal
if __name__ == "__main__":
  print("P NZ  fwd wavefronts (NB=2 + NB=1) unpadded -> (best, PER, ZS, YS, FPAD) | inv unpadded -> (best, DS, ES)")
  for P in (3,4,5,6,7,8,10,12):
      NG = 2*P-1; NZ = NG//2+1
      base = fwd_cost(P, NZ, NZ)
      cands = []
      for ZS in range(NZ, NZ+9):
          for YS in range(NZ, NZ+9):
              for PAD in (0, 2, 4, 8):
                  c, i, per = fwd_cost(P, ZS, YS, 2, PAD)
                  c1, _, _ = fwd_cost(P, ZS, YS, 1, PAD)
                  cands.append((c + c1, per, ZS, YS, PAD))
      best = min(cands)
      ib = inv_cost(P, NZ, NZ)
      ibest = min(((inv_cost(P, DS, ES)[0], DS, ES) for DS in range(NZ, NZ+9) for ES in range(NZ, NZ+9)))
      print(P, "NZ", NZ, "fwd(nbc2+nbc1) base", fwd_cost(P,NZ,NZ,2)[0]+fwd_cost(P,NZ,NZ,1)[0], "best", best, "| inv base", ib[0], "best", ibest)
