// Fast walker of k_sched_round<BM> (BM = 1 or 4): beam_schedule
// (scheduler.cpp:289-378) for beam width B <= BM over at most 8 engine pools
// with at most 255 free slots each -- the shapes of BASELINE config 3 (B in
// {1, 4}, 8 pools) and of the shipped scenarios.  Textually included into the
// walker branch of k_sched_round (ag_sched.cu); the general walker there
// covers every other shape.
//
// Nested retention (scheduler.cpp:351-370) can only adopt the best B - p
// children of parent p, so a step needs at most B(B+1)/2 "relevant"
// children (10 for B = 4).  Lane c is relevant child k of parent p (lanes
// 0-3: parent 0, 4-6: parent 1, 7-8: parent 2, 9: parent 3) and holds a copy
// of BeamState p (util, flex sum/count, skips, last history node, path
// length, free-engine mask, one free-slot byte per engine).  A step:
//   * the next candidate: one ballot over the next 32 entries of the
//     lookahead ring (records, engine masks and histogram rows fetched ahead
//     by warp 1) against the union of free masks;
//   * allowed_engines (scheduler.cpp:140-156): the candidate's engine mask &
//     the state's free mask (a re-touch -- a request with parallel ready
//     branches -- counts survivors over the viable list instead);
//   * lane (p, k) builds child k of p from the k-th allowed engine (engines
//     are in weight-descending order, so util + w_e is non-increasing along
//     the mask: the first B - p set bits are p's best children unless the
//     boundary ties in utilization -- then p's children are sorted exactly
//     first): utilization, flexibility, skips and the extend_state deltas
//     (scheduler.cpp:158-206);
//   * every relevant child ranks itself against the others under the exact
//     state_better order, read as (util, flexibility, skips, lex key) from
//     shared memory.  The lex key orders triples_less exactly: while the walk
//     visits requests in increasing request index every triple already in a
//     list precedes the new one, so the children's order is the parents'
//     order (from the relation table and whether the parent has only its
//     skip child, which a prefix relation decides) and then the model; a
//     re-touch or a non-monotone container order ranks the lists pairwise;
//   * nested retention is then bit arithmetic: level w takes the lowest rank
//     not yet taken among the rank masks of parents < w;
//   * lanes of group w copy pick w (shuffles from the picked child's lane);
//     the picked lanes append history nodes; lanes (w1, w2) update the
//     triples_less relations of the new beam.
// The beam leaves in the general walker's lane layout (state w in lane w,
// occupancy rows in s_occ) for the common finalize.
{
  constexpr int kB = BM;
  constexpr int kRel = kB * (kB + 1) / 2;  // relevant children (lanes)
  // first lane of group (parent) p, and the group of lane c
  auto group_start = [](int p) -> int { return p * kB - p * (p - 1) / 2; };
  auto group_of = [&](int c) -> int {
    int p = 0;
#pragma unroll
    for (int q = 0; q < kB; ++q)
      if (c >= group_start(q + 1)) p = q + 1;
    return p;
  };
  const int gp = lane < kRel ? group_of(lane) : kB;  // kB: not a relevant lane
  const int gk = lane < kRel ? lane - group_start(gp) : 0;
  const bool lead = lane < kRel && gk == 0;  // first lane of its group
  // Pairwise ranking: the kRel(kRel-1)/2 unordered pairs (i < j) of relevant
  // children, pair t in lane t % 32 of round t / 32; a round's ballot holds
  // "j is better than i" per pair.  Lane c's rank is then four popcounts
  // over the ballots with its constant masks: pairs (c, j) where j is better,
  // pairs (j, c) where c is not.
  constexpr int kPairs = kRel * (kRel - 1) / 2;
  int pi0 = 0, pj0 = 0, pi1 = 0, pj1 = 0;  // my pairs of rounds 0 and 1
  uint32_t gt0 = 0, gt1 = 0, lt0 = 0, lt1 = 0;
  {
    int t = 0;
    for (int i = 0; i < kRel; ++i)
      for (int jj = i + 1; jj < kRel; ++jj, ++t) {
        const uint32_t bit = 1u << (t & 31);
        if (t == lane) pi0 = i, pj0 = jj;
        if (t == lane + 32) pi1 = i, pj1 = jj;
        if (i == lane) (t < 32 ? gt0 : gt1) |= bit;
        if (jj == lane) (t < 32 ? lt0 : lt1) |= bit;
      }
  }
  // packed group of each relevant lane (4 bits per lane, lanes < 16)
  constexpr unsigned long long kGroupTab = [] {
    unsigned long long t = 0;
    int c = 0;
    for (int p = 0; p < kB; ++p)
      for (int k = 0; k < kB - p; ++k, ++c) t |= (unsigned long long)p << (4 * c);
    return t;
  }();
  // relation masks of the current beam (bit q * kB + p: rel[q][p] is LESS /
  // P1 / P2), rebuilt by ballots after every step
  uint32_t rel_less = 0, rel_p1 = 0, rel_p2 = 0;
  // free slots per engine, one byte each (the host guarantees <= 255)
  auto free_bytes = [&]() -> uint64_t {
    uint64_t r = 0;
    for (int e = 0; e < E; ++e) {
      const int fr = e_slots[e] - A.eng.occ[e];
      r |= (uint64_t)(fr > 0 ? (fr < 255 ? fr : 255) : 0) << (8 * e);
    }
    return r;
  };
  // lane c: a copy of BeamState gp (lane 0 computed initial_state above)
  double u = __shfl_sync(kFull, st_u, 0), fs = 0.0;
  int fc = 0, sk = 0, nd = -1, ln = 0;
  uint32_t fm = __shfl_sync(kFull, st_fm, 0);
  uint64_t rem = free_bytes();
  const double* const sw = e_weight;
  // a request's pairs are consecutive in the two-level order and history
  // nodes are numbered in creation order, so a state touched the current
  // request iff its last node was created since the walk reached it
  int q_last = -1, q_node0 = 0;
  int q_prev = -1;  // largest request index visited so far

  // the next candidate whose engine mask meets a free engine of U, from the
  // lookahead ring (records, masks and histogram rows already in shared
  // memory): one ballot over the next 32 ring entries; le = its ring slot.
  // The walker's union and consumed count are published for the lookahead.
  const int LA = A.la_rows;
  unsigned la_tail = 0, la_head = 0;
  auto ring_next = [&](uint32_t U, int& le, uint32_t& base) -> bool {
    if (lane == 0) {
      *(volatile uint32_t*)&s_U = U;
      st_release(&s_la_tail, la_tail);  // entries before it are no longer read
    }
    for (;;) {
      if (la_tail == la_head) {
        unsigned h = 0;
        if (lane == 0) {
          // every entry so far is consumed (skipped ones included): the
          // lookahead must see the room before it can refill the ring
          st_release(&s_la_tail, la_tail);
          for (;;) {
            const unsigned done = *(volatile unsigned*)&s_la_done;
            h = *(volatile unsigned*)&s_la_head;
            if (h > la_tail || done) break;
          }
          h = ld_acquire(&s_la_head);
        }
        la_head = __shfl_sync(kFull, h, 0);
        if (la_head == la_tail) return false;  // list exhausted
      }
      const unsigned i = la_tail + (unsigned)lane;
      const uint32_t m = i < la_head ? s_la_mask[i & (unsigned)(LA - 1)] : 0u;
      const unsigned b = __ballot_sync(kFull, (m & U) != 0u);
      if (b) {
        const int src = __ffs(b) - 1;
        le = (int)((la_tail + (unsigned)src) & (unsigned)(LA - 1));
        base = __shfl_sync(kFull, m, src);
        la_tail += (unsigned)src + 1u;
        return true;
      }
      la_tail = min(la_head, la_tail + 32u);
    }
  };
  // re-touch of state si (last node snode): counts per model of this agent
  // over the request's viable configurations consistent with the state's
  // earlier triples for it (s_cnt[si]), the flex delta per model surv /
  // initial - before (extend_state :196-203; s_rdelta[si]); returns the
  // engine mask of the models with survivors
  auto retouch = [&](int si, int snode, int qcur, int a, int slot, double initial) -> uint32_t {
    if (lane == 0) {
      int n = snode, nc = 0;
      while (n >= 0 && nv[n].qi == qcur) {
        s_cons[nc][0] = nv[n].am >> 8;
        s_cons[nc][1] = nv[n].am & 0xFF;
        ++nc;
        n = nv[n].prev;
      }
      s_ncons = nc;
    }
    s_cnt[si][lane] = 0;
    __syncwarp();
    const int ncons = s_ncons;
    const uint32_t* vl = A.pool + A.voff[slot];
    const uint32_t nv_len = A.nviable[slot];
    for (uint32_t q = lane; q < nv_len; q += 32) {
      const uint32_t c = vl[q];
      bool ok = true;
      for (int t = 0; t < ncons && ok; ++t) ok = (int)digit_at(c, s_cons[t][0], A) == s_cons[t][1];
      if (ok) atomicAdd(&s_cnt[si][digit_at(c, a, A)], 1);
    }
    __syncwarp();
    uint32_t em = 0;
    for (int m2 = 0; m2 < M; ++m2)
      if (s_cnt[si][m2] > 0) em |= 1u << e_m2e[m2];
    if (lane < M) {
      const int before = snode >= 0 ? nv[snode].nsurv : 0;
      s_rdelta[si][lane] = (double)s_cnt[si][lane] / initial - (double)before / initial;
    }
    __syncwarp();
    return em;
  };

  if constexpr (kB == 1) {
    // Beam width 1: one state (uniform in every lane) and no retention: a
    // candidate with a free allowed engine takes the state's best child --
    // the heaviest such engine, unless the next one ties in utilization
    // (then flexibility, then model decide) -- otherwise every pair is a skip.
    while (!wstatus && fm) {
      int le = 0;
      uint32_t base = 0;
      const bool got = ring_next(fm, le, base);
      AG_PHASE_TICK(0);
      if (!got) break;
      const Cand cr = s_la_rec[le];
      if ((long long)cr.pos > pi) {
        sk += (int)((long long)cr.pos - pi);
        explored += (unsigned long long)((long long)cr.pos - pi);
      }
      pi = (long long)cr.pos + 1;
      const int qcur = cr.qi, a = (int)(cr.slot_agent >> 26), slot = (int)(cr.slot_agent & 0x3ffffffu);
      const double initial = (double)cr.nvia;
      if (qcur != q_last) q_last = qcur, q_node0 = nnodes;
      const bool touched = nd >= q_node0;
      uint32_t mk = base & fm;
      if (__builtin_expect(touched, 0)) mk = retouch(0, nd, qcur, a, slot, initial) & fm;
      if (!mk) {  // whole-beam skip
        sk += 1;
        explored += 1;
        continue;
      }
      explored += (unsigned long long)__popc(mk);
      ++n_steps;
      auto delta_of = [&](int m) -> double { return touched ? s_rdelta[0][m] : h_rat[le * M + m]; };
      int e = __ffs(mk) - 1;
      double cu = u + sw[e];
      const uint32_t after = mk & ~((2u << e) - 1u);
      if (__builtin_expect(after && u + sw[__ffs(after) - 1] == cu, 0)) {
        // equal utilizations: state_better's flexibility, then the model
        double bf = 0.0;
        int be = -1;
        for (uint32_t t = mk; t; t &= t - 1) {
          const int ee = __ffs(t) - 1;
          const double x = u + sw[ee];
          if (x != cu) continue;
          const double xf = (fs + delta_of(e_model[ee])) / (touched ? fc : fc + 1);
          if (be < 0 || xf > bf || (xf == bf && e_model[ee] < e_model[be])) be = ee, bf = xf;
        }
        e = be;
      }
      AG_PHASE_TICK(1);
      const int mdl = e_model[e];
      const uint32_t sv = touched ? (uint32_t)s_cnt[0][mdl] : h_cnt[le * M + mdl];
      if (nnodes + 1 > A.max_nodes) {
        wstatus = AG_ERR_INTERNAL + 300;  // history overflow
        break;
      }
      if (lane == 0) {
        Node n;
        n.qi = qcur;
        n.am = (a << 8) | mdl;
        n.prev = nd;
        n.depth = ln + 1;
        n.nsurv = (int)sv;
        n.nvia = cr.nvia;
        n.slot = slot;
        n.pad = 0;
        if (nnodes < kSmemNodes) s_nodes[nnodes] = n;
        else A.gnodes[nnodes - kSmemNodes] = n;
      }
      u = cu;
      fs += delta_of(mdl);
      fc += touched ? 0 : 1;
      rem -= 1ull << (8 * e);
      if (!((rem >> (8 * e)) & 0xffull)) fm &= ~(1u << e);
      nd = nnodes++;
      ++ln;
      AG_PHASE_TICK(3);
    }
    __syncwarp();
  } else
  while (!wstatus) {
    const bool live = gp < nst;  // my group's state exists
    const uint32_t U = __reduce_or_sync(kFull, lead && live ? fm : 0u);
    if (!U) break;  // all-full early exit (scheduler.cpp:303-315)
    int le = 0;
    uint32_t base = 0;
    const bool got = ring_next(U, le, base);
    AG_PHASE_TICK(0);
    if (!got) break;
    const Cand cr = s_la_rec[le];
    {  // whole-beam skips before this pair
      const long long k = (long long)cr.pos - pi;
      if (k > 0) {
        if (live) sk += (int)k;
        explored += (unsigned long long)nst * (unsigned long long)k;
      }
      pi = (long long)cr.pos + 1;
    }
    const int qcur = cr.qi, a = (int)(cr.slot_agent >> 26), slot = (int)(cr.slot_agent & 0x3ffffffu);
    const double initial = (double)cr.nvia;
    const uint64_t key_base = tkey(qcur, a, 0);
    if (qcur != q_last) q_last = qcur, q_node0 = nnodes;
    // ---- allowed_engines (every lane of group p: state p)
    const bool touched = live && nd >= q_node0;
    uint32_t mk = live ? (base & fm) : 0u;
    const uint32_t tlead = __ballot_sync(kFull, lead && touched);  // bit group_start(p)
    if (tlead) {
      // re-touch: counts per model of this agent over the request's viable
      // configurations consistent with the state's earlier triples for it
      for (uint32_t tb = tlead; tb; tb &= tb - 1) {
        const int sl = __ffs(tb) - 1, si = group_of(sl);
        const uint32_t em = retouch(si, __shfl_sync(kFull, nd, sl), qcur, a, slot, initial);
        if (gp == si) mk = em & fm;
      }
    }
    if (!__any_sync(kFull, mk != 0u)) {  // whole-beam skip (scheduler.cpp:317-329)
      if (live) sk += 1;
      explored += (unsigned long long)nst;
      continue;
    }
    explored += (unsigned long long)__reduce_add_sync(kFull, lead && live ? (mk ? __popc(mk) : 1u) : 0u);
    ++n_steps;
    // flex_sum delta of a child on model m: the first-touch ratio surv /
    // initial (fetched by the lookahead), or the re-touch delta computed above
    auto delta_of = [&](int m) -> double { return touched ? s_rdelta[gp][m] : h_rat[le * M + m]; };
    // ---- my child: the gk-th allowed engine of state gp (or its skip child)
    const int nall = __popc(mk);
    const bool valid = live && (mk ? gk < nall : gk == 0);
    int e = -1;
    {
      uint32_t m1 = mk;
#pragma unroll
      for (int k = 0; k + 1 < kB; ++k)
        if (gk > k) m1 &= m1 - 1;
      if (valid && m1) e = __ffs(m1) - 1;
    }
    double cu = e >= 0 ? u + sw[e] : u;
    // boundary: the parent's next child beyond its B - p relevant ones ties
    // with the last relevant one -- then the group's children are sorted
    // exactly (util desc, flexibility desc, model asc: siblings share skips
    // and differ in the last triple only)
    const uint32_t after = e >= 0 ? mk & ~((2u << e) - 1u) : 0u;  // allowed engines after mine
    const bool bnd = valid && e >= 0 && gk == kB - 1 - gp && after && u + sw[__ffs(after) - 1] == cu;
    const uint32_t bmask = __ballot_sync(kFull, bnd);
    if (bmask) {
      for (uint32_t tb = bmask; tb; tb &= tb - 1) {
        const int gsrc = group_of(__ffs(tb) - 1);
        if (lane == group_start(gsrc)) {
          uint32_t rm = mk;
          for (int k = 0; k < kB - gsrc && rm; ++k) {
            int be = -1;
            double bu = 0.0, bf = 0.0;
            for (uint32_t t = rm; t; t &= t - 1) {
              const int ee = __ffs(t) - 1;
              const double x = u + sw[ee];
              const double xf = (fs + delta_of(e_model[ee])) / (touched ? fc : fc + 1);
              if (be < 0 || x > bu || (x == bu && (xf > bf || (xf == bf && e_model[ee] < e_model[be]))))
                be = ee, bu = x, bf = xf;
            }
            rm &= ~(1u << be);
            s_order[gsrc][k] = (int8_t)be;
          }
        }
        __syncwarp();
        if (gp == gsrc && valid) {
          e = s_order[gsrc][gk];
          cu = u + sw[e];
        }
        __syncwarp();
      }
    }
    // the child's extend_state deltas; its flexibility is state_better's
    // second key
    const int mdl = e >= 0 ? e_model[e] : 0;
    const double nfs = e >= 0 ? fs + delta_of(mdl) : fs;
    const int nfc = e >= 0 && !touched ? fc + 1 : fc;
    const double cf = nfc > 0 ? nfs / nfc : 1.0;
    const int cs = e >= 0 ? sk : sk + 1;
    AG_PHASE_TICK(1);
    // ---- the lex key of my child (triples_less among the relevant children)
    const uint32_t V = __ballot_sync(kFull, valid);
    int lexkey;
    if (__builtin_expect(qcur > q_prev, 1)) {
      // every existing triple precedes the new key: the order of parent q's
      // children before parent p's depends on rel[q][p] and, for a prefix
      // relation, on whether the shorter list's parent only has its skip child
      const uint32_t skip_only = __ballot_sync(kFull, lead && live && mk == 0u);
      uint32_t qskip = 0;  // bit q: parent q only has its skip child
#pragma unroll
      for (int q = 0; q < kB; ++q) qskip |= ((skip_only >> group_start(q)) & 1u) << q;
      const bool p_skip = (qskip >> (gp & (kB - 1))) & 1u;
      int prank = 0;
#pragma unroll
      for (int q = 0; q < kB; ++q) {
        const int bit = q * kB + (gp & (kB - 1));
        prank += ((rel_less >> bit) & 1u) | ((rel_p1 >> bit) & (qskip >> q) & 1u) |
                 ((rel_p2 >> bit) & 1u & (uint32_t)!p_skip);
      }
      lexkey = prank * 64 + (e >= 0 ? mdl + 1 : 0);
    } else {
      // exact pairwise triples_less (a re-touch, or requests out of index order)
      if (lane < kRel) s_fe[lane] = (int8_t)e;
      __syncwarp();
      lexkey = 0;
      if (valid) {
        const uint64_t mykey = e >= 0 ? key_base | (uint64_t)(uint32_t)mdl : kEnd;
        for (int c = 0; c < kRel; ++c) {
          if (c == lane || !((V >> c) & 1u)) continue;
          const int pc = group_of(c), ec = s_fe[c];
          const uint64_t ck = ec >= 0 ? key_base | (uint64_t)(uint32_t)e_model[ec] : kEnd;
          lexkey += lex_before(pc == gp, s_rel[cur][pc][gp], ck, mykey);
        }
      }
    }
    q_prev = qcur > q_prev ? qcur : q_prev;
    // ---- exact rank of my child among the relevant children: state_better
    // on (util desc, flexibility desc, skips asc, lex key asc), branch-free
    if (lane < kRel) {
      s_fkey[lane] = valid ? make_double2(cu, cf) : make_double2(-INFINITY, -INFINITY);
      s_fmeta[lane] = valid ? ((unsigned long long)(uint32_t)cs << 16) | (unsigned)lexkey : ~0ull;
    }
    __syncwarp();
    auto better = [&](int i, int jj) -> bool {  // child jj before child i (state_better)
      const double2 ki = s_fkey[i], kj = s_fkey[jj];
      const unsigned long long mi = s_fmeta[i], mj = s_fmeta[jj];
      return kj.x > ki.x || (kj.x == ki.x && (kj.y > ki.y || (kj.y == ki.y && mj < mi)));
    };
    const uint32_t b0 = __ballot_sync(kFull, lane < kPairs && better(pi0, pj0));
    const uint32_t b1 = kPairs > 32 ? __ballot_sync(kFull, lane + 32 < kPairs && better(pi1, pj1)) : 0u;
    const int rank = __popc(b0 & gt0) + __popc(b1 & gt1) + __popc(~b0 & lt0) + __popc(~b1 & lt1);
    AG_PHASE_TICK(2);
    // ---- nested retention: level w adopts the lowest rank not yet taken
    // among the rank masks of parents < w
    uint32_t Rm[kB];
#pragma unroll
    for (int p = 0; p < kB; ++p) Rm[p] = __reduce_or_sync(kFull, valid && gp == p ? 1u << rank : 0u);
    int src[kB], pe[kB];
    int npick = 0;
    uint32_t avail = 0, taken = 0;
#pragma unroll
    for (int w = 0; w < kB; ++w) {
      src[w] = 0;
      if (w >= B) continue;
      avail |= Rm[w];
      const uint32_t av = avail & ~taken;
      if (!av) continue;
      const int r = __ffs(av) - 1;
      taken |= 1u << r;
      src[w] = __ffs(__ballot_sync(kFull, valid && rank == r)) - 1;
      npick = w + 1;
    }
    int pp[kB], ebef[kB + 1];  // parent of pick w; engine picks before level w
    ebef[0] = 0;
#pragma unroll
    for (int w = 0; w < kB; ++w) {
      pe[w] = __shfl_sync(kFull, e, src[w]);
      pp[w] = (int)((kGroupTab >> (4 * src[w])) & 0xFull);
      ebef[w + 1] = ebef[w] + (w < npick && pe[w] >= 0);
    }
    const int eng_before = ebef[kB];
    // ---- adoption: group w copies pick w; the picked lane appends the node
    int my_src = src[0], my_id = nnodes, my_w = -1;
#pragma unroll
    for (int w = 0; w < kB; ++w) {
      if (w < npick && gp == w) my_src = src[w], my_id = nnodes + ebef[w];
      if (w < npick && lane == src[w]) my_w = w;
    }
    if (my_w >= 0 && e >= 0 && !wstatus) {
      int id = nnodes;
#pragma unroll
      for (int w = 1; w < kB; ++w)
        if (my_w == w) id = nnodes + ebef[w];
      if (id < A.max_nodes) {
        Node n;
        n.qi = qcur;
        n.am = (a << 8) | mdl;
        n.prev = nd;
        n.depth = ln + 1;
        n.nsurv = (int)(touched ? (uint32_t)s_cnt[gp][mdl] : h_cnt[le * M + mdl]);
        n.nvia = cr.nvia;
        n.slot = slot;
        n.pad = 0;
        if (id < kSmemNodes) s_nodes[id] = n;
        else A.gnodes[id - kSmemNodes] = n;
      }
    }
    if (nnodes + eng_before > A.max_nodes) wstatus = AG_ERR_INTERNAL + 300;  // history overflow (uniform)
    {
      const uint64_t crem = e >= 0 ? rem - (1ull << (8 * e)) : rem;
      const uint32_t cfm = e >= 0 && !((crem >> (8 * e)) & 0xffull) ? fm & ~(1u << e) : fm;
      const double a_u = __shfl_sync(kFull, cu, my_src), a_fs = __shfl_sync(kFull, nfs, my_src);
      const int a_fc = __shfl_sync(kFull, nfc, my_src), a_sk = __shfl_sync(kFull, cs, my_src);
      const int a_nd = __shfl_sync(kFull, nd, my_src), a_ln = __shfl_sync(kFull, ln, my_src);
      const int a_e = __shfl_sync(kFull, e, my_src);
      const uint32_t a_fm = __shfl_sync(kFull, cfm, my_src);
      const uint64_t a_rem = __shfl_sync(kFull, crem, my_src);
      if (gp < npick) {
        u = a_u, fs = a_fs, fc = a_fc, sk = a_sk, fm = a_fm, rem = a_rem;
        nd = a_e >= 0 ? my_id : a_nd;
        ln = a_e >= 0 ? a_ln + 1 : a_ln;
      }
    }
    nnodes += eng_before;
    // ---- triples_less relations of the new beam: lane (w1, w2) per ordered pair
    if constexpr (kB > 1) {
      const int nxt = cur ^ 1;
      const int w1 = lane / kB, w2 = lane % kB;
      int p1 = pp[0], p2 = pp[0], e1 = pe[0], e2 = pe[0];
#pragma unroll
      for (int q = 1; q < kB; ++q) {
        if (w1 == q) p1 = pp[q], e1 = pe[q];
        if (w2 == q) p2 = pp[q], e2 = pe[q];
      }
      uint64_t code = kRelGreater;
      if (lane < kB * kB && w1 < npick && w2 < npick && w1 != w2) {
        const uint64_t k1 = e1 < 0 ? kEnd : key_base | (uint64_t)(uint32_t)e_model[e1];
        const uint64_t k2 = e2 < 0 ? kEnd : key_base | (uint64_t)(uint32_t)e_model[e2];
        const uint64_t r12 = p1 != p2 ? s_rel[cur][p1][p2] : 0ull;
        const uint64_t r = rel_extend_sel(p1 == p2, r12, k1, k2);
        s_rel[nxt][w1][w2] = r;
        code = r & kRelCode;
      }
      rel_less = __ballot_sync(kFull, code == kRelLess);
      rel_p1 = __ballot_sync(kFull, code == kRelP1);
      rel_p2 = __ballot_sync(kFull, code == kRelP2);
      cur = nxt;
    }
    nst = npick;
    __syncwarp();
    AG_PHASE_TICK(3);
  }
  __syncwarp();
  // hand the beam to the common finalize: state w in lane w, occupancy rows
  {
    const int from = group_start(lane < kB ? lane : 0);
    const double x_u = __shfl_sync(kFull, u, from), x_fs = __shfl_sync(kFull, fs, from);
    const int x_fc = __shfl_sync(kFull, fc, from), x_sk = __shfl_sync(kFull, sk, from);
    const int x_nd = __shfl_sync(kFull, nd, from), x_ln = __shfl_sync(kFull, ln, from);
    st_u = x_u, st_fs = x_fs, st_fc = x_fc, st_sk = x_sk, st_nd = x_nd, st_ln = x_ln;
    const int w = lane >> 3, ee = lane & 7;
    const uint64_t r = __shfl_sync(kFull, rem, group_start(w < kB ? w : 0));
    if (w < nst && ee < E)
      s_occ[cur][w][ee] = A.eng.occ[ee] + (int)((free_bytes() >> (8 * ee)) & 0xffull) - (int)((r >> (8 * ee)) & 0xffull);
  }
  __syncwarp();
}
