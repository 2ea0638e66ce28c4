// baselines.cuh — the reference's comparison policies (engine.hpp:383-726):
// Orca, vLLM, Sarathi, MultiRes and SyncCoupled, on the same per-instance
// device structures as the econoserve family (included by engine.cuh).
//
//   wait_fifo_ (engine.hpp:1023)  -> the FIFO min tree over request ids: the
//       FIFO only ever holds a sorted id set (arrivals append in id order,
//       preemptions re-insert at lower_bound, E:477-479 / E:924-926), so
//       "front" is the first present leaf. Leaves hold the request's
//       forward-size demand (prompt, or 1 once it has generated), which
//       MultiRes' scan prunes on. I.pt_count is the FIFO's size.
//   waiting_groups_ (E:1022)     -> the GT group queue (sync-coupled only;
//       the econoserve gt_queue_ is unused by these policies).
//   admit_order_ (E:1025)        -> I.admo, ongoing_prefills_ (E:1024) ->
//       I.ongo: short ordered id lists (bounded by the running set).
//   prefill_target (request.hpp) -> I.ptarget (recompute preemption moves it).
// Block grants (kvc.hpp:134-142) are one-block regions from the same
// first-fit allocator as exact allocations.
#pragma once

// std::erase of an id from an ordered id list (the lists hold unique ids).
EDEV void list_erase(GP<int32_t> a, int32_t* n, int32_t v) {
  const int32_t pos = arr_find(a, *n, v);
  if (pos < 0) return;
  arr_erase(a, *n, pos, 1);
  LANE0((*n)--);
}

// ---- wait_fifo_ ----
EDEV void wait_insert(Inst& I, int32_t id) {
  const int32_t gpu = I.generated[id] > 0 ? 1 : I.prompt[id];
  tree_set(I, id, gpu);
  LANE0(I.pt_count++);
}
EDEV int32_t wait_front(const Inst& I) { return I.pt_count > 0 ? tree_first(I, 0, INF32 - 1) : -1; }
EDEV void wait_remove(Inst& I, int32_t id) {
  tree_set(I, id, INF32);
  LANE0(I.pt_count--);
}

// allocate_block (kvc.hpp:134-142)
EDEV bool alloc_block(Inst& I, int32_t id) { return kvc_alloc_region(I, id, I.block); }

// lifo_victim (engine.hpp:447-455): most recently admitted running request
// other than `exclude`, scanning admit_order_ from the back W at a time.
EDEV int32_t lifo_victim(const Inst& I, int32_t exclude) {
  for (int32_t hi = I.n_admo - 1; hi >= 0; hi -= W) {
    const int32_t j = hi - LANE;
    int32_t id = -1;
    bool ok = false;
    if (j >= 0) {
      id = I.admo[j];
      ok = id != exclude && I.state[id] == ST_RUNNING;
    }
    const unsigned m = BALLOT(ok);
    if (m) return shfl(id, FFS(m));
  }
  return -1;
}

// Waiting/preemption-time accrual shared by resume_decode / resume_prefill
// (engine.hpp:408-414, 546-551), lane 0.
EDEV void accrue_wait(Inst& I, int32_t id) {
  const uint8_t f = I.flags[id];
  const double le = I.last_enq[id], wt = I.waiting[id], pt = I.preempt_t[id];
  const double wait = dmax(0.0, I.clock - le);
  if (f & F_WAS_PREEMPTED) I.preempt_t[id] = pt + wait; else I.waiting[id] = wt + wait;
  I.flags[id] = (uint8_t)(f & ~F_WAS_PREEMPTED);
  I.state[id] = ST_RUNNING;
}
// resume_decode (engine.hpp:407-420)
EDEV void resume_decode(Inst& I, int32_t id) {
  if (LANE == 0) {
    accrue_wait(I, id);
    I.gen_epoch[id] = I.generated[id];
    I.run[I.R++] = id;
    I.adm[I.n_adm++] = id;
    I.admo[I.n_admo++] = id;
  }
  WSYNC();
}
// resume_prefill (engine.hpp:545-556)
EDEV void resume_prefill(Inst& I, int32_t id, Tok chunk) {
  if (LANE == 0) {
    accrue_wait(I, id);
    I.ptiter_id[I.n_ptiter] = id;
    I.ptiter_tok[I.n_ptiter] = (int32_t)chunk;
    I.n_ptiter++;
    I.adm[I.n_adm++] = id;
    I.admo[I.n_admo++] = id;
  }
  WSYNC();
}
// dispatch_pt_common (engine.hpp:372-381)
EDEV void dispatch_common(Inst& I, int32_t id, Tok tokens) {
  if (LANE == 0) {
    const double arr = I.arrival[id], wt = I.waiting[id];
    I.state[id] = ST_RUNNING;
    I.dispatch_t[id] = I.clock;
    I.waiting[id] = wt + (I.clock - arr);
    I.ptiter_id[I.n_ptiter] = id;
    I.ptiter_tok[I.n_ptiter] = (int32_t)tokens;
    I.n_ptiter++;
    I.adm[I.n_adm++] = id;
    I.admo[I.n_admo++] = id;
    I.pts_admitted_iter++;
    I.pt_dispatched++;
  }
  WSYNC();
  logev(I, ECONO_EV_PT_DISPATCH, id, 0, 0);
  WSYNC();
}
// kvc_.add_written (kvc.hpp:87-90) for a swap-in and the occupied count, lane 0.
EDEV void swap_in(Inst& I, int32_t id, Tok restored) {
  LANE0(const int32_t wr = I.written[id]; I.written[id] = (int32_t)restored;
        I.written_total += restored - wr; I.occupied[id] = (int32_t)restored;
        I.pending_stall += I.swap_stall);
  logev(I, ECONO_EV_SWAP_IN, id, 0, 0);
  WSYNC();
}

// preempt_swap (engine.hpp:458-481)
EDEVNI void preempt_swap(Inst& I, int32_t id) {
  const Tok w = I.written[id];
  kvc_release(I, id);
  if (I.error) return;
  if (LANE == 0) {
    const int32_t gen = I.generated[id], pr = I.prompt[id];
    I.occupied[id] = 0;
    I.preempt_count[id]++;
    I.state[id] = ST_PREEMPTED;
    I.flags[id] |= F_WAS_PREEMPTED;
    I.last_enq[id] = I.clock;
    if (I.recompute) {
      I.prefill_done[id] = 0;
      I.ptarget[id] = pr + gen;
    }
  }
  WSYNC();
  list_erase(I.run, &I.R, id);
  list_erase(I.admo, &I.n_admo, id);
  list_erase(I.ongo, &I.n_ongo, id);
  const int32_t pos = arr_find(I.ptiter_id, I.n_ptiter, id);
  if (pos >= 0) {
    arr_erase(I.ptiter_id, I.n_ptiter, pos, 1);
    arr_erase(I.ptiter_tok, I.n_ptiter, pos, 1);
    LANE0(I.n_ptiter--);
  }
  wait_insert(I, id);
  logev(I, ECONO_EV_PREEMPT_SWAP, id, w, 0);
  WSYNC();
}

// Block-grant failure bookkeeping (engine.hpp:434-439, 636-642).
EDEV void note_alloc_fail(Inst& I, int32_t id) {
  LANE0(I.flags[id] |= F_ALLOC_FAIL; I.alloc_failures++);
  logev(I, ECONO_EV_ALLOC_FAIL, id, 0, 0);
  WSYNC();
}

// ensure_blocks_for (engine.hpp:630-653)
EDEVNI bool ensure_blocks_for(Inst& I, int32_t id, Tok resident) {
  const Tok need = block_round(resident, I.block);
  bool flagged = false;
  while ((Tok)I.held[id] < need) {
    if (alloc_block(I, id)) continue;
    if (I.error) return false;
    if (!flagged) {
      flagged = true;
      note_alloc_fail(I, id);
    }
    const int32_t victim = lifo_victim(I, id);
    if (victim < 0) {
      preempt_swap(I, id);
      return false;
    }
    preempt_swap(I, victim);
    if (I.error || I.state[id] != ST_RUNNING) return false;
  }
  return true;
}

// grow_decode_blocks (engine.hpp:426-445). Candidates (running, nothing left
// of their last block) are fixed by one pass in running order: processing a
// candidate only changes its own holdings or preempts a victim, which the
// state test then skips, so no other request's test outcome can change.
EDEVNI void grow_decode_blocks(Inst& I) {
  int32_t nc = 0;
  for (int32_t base = 0; base < I.R; base += W) {
    const int32_t i = base + LANE;
    bool c = false;
    int32_t id = -1;
    if (i < I.R) {
      id = I.run[i];
      c = I.state[id] == ST_RUNNING && I.held[id] - I.written[id] < 1;
    }
    const unsigned m = BALLOT(c);
    if (c) I.cd_ri[nc + POPC(m & LANEMASK_LT)] = id;
    nc += POPC(m);
  }
  WSYNC();
  for (int32_t k = 0; k < nc; ++k) {
    const int32_t id = I.cd_ri[k];
    if (I.state[id] != ST_RUNNING) continue;
    bool flagged = false;
    while (!alloc_block(I, id)) {
      if (I.error) return;
      if (!flagged) {
        flagged = true;
        note_alloc_fail(I, id);
      }
      const int32_t victim = lifo_victim(I, id);
      if (victim < 0) {
        preempt_swap(I, id);
        break;
      }
      preempt_swap(I, victim);
      if (I.error) return;
    }
    if (I.error) return;
  }
}

// The prefills of this iteration claim the blocks for the tokens they will
// write, over a copy of pt_iter_ (engine.hpp:526-532, 623-627).
EDEVNI void claim_prefill_blocks(Inst& I) {
  const int32_t np = I.n_ptiter;
  for (int32_t i = LANE; i < np; i += W) {
    I.cd_abs[i] = I.ptiter_id[i];
    I.cd_use[i] = I.ptiter_tok[i];
  }
  WSYNC();
  for (int32_t k = 0; k < np; ++k) {
    const int32_t id = I.cd_abs[k];
    if (I.state[id] != ST_RUNNING) continue;
    ensure_blocks_for(I, id, (Tok)I.prefill_done[id] + I.cd_use[k]);
    if (I.error) return;
  }
}

// form_orca (engine.hpp:386-405): FCFS, max-allocation, batch cap.
EDEVNI void form_orca(Inst& I) {
  while (I.pt_count > 0) {
    const int32_t active = I.R + I.n_ptiter + I.n_ongo;
    if (active >= I.batch_cap) break;
    const int32_t id = wait_front(I);
    LANE0(I.exam_count++);
    const Tok need = (Tok)I.prompt[id] + I.max_out;
    if (I.held[id] > 0) {  // resumed after a preemption: space is still held
      wait_remove(I, id);
      LANE0(I.allowance[id] = (int32_t)I.max_out);
      resume_decode(I, id);
      continue;
    }
    if (!kvc_alloc_region(I, id, need)) break;  // strict FCFS head-of-line
    if (I.error) return;
    LANE0(I.allowance[id] = (int32_t)I.max_out);
    wait_remove(I, id);
    dispatch_common(I, id, I.prompt[id]);
  }
}

// form_vllm (engine.hpp:483-543)
EDEVNI void form_vllm(Inst& I) {
  grow_decode_blocks(I);
  if (I.error) return;
  Tok prompts = 0;
  while (I.pt_count > 0) {
    const int32_t id = wait_front(I);
    LANE0(I.exam_count++);
    const Tok pdone = I.prefill_done[id], ptg = I.ptarget[id], pr = I.prompt[id], gen = I.generated[id];
    const Tok held = I.held[id];
    const double dsp = I.dispatch_t[id];
    const Tok prefill_tokens = pdone < ptg ? ptg - pdone : 0;
    const Tok decodes = I.R;
    if (prefill_tokens > 0 && decodes + prompts + prefill_tokens > I.tfs && (prompts > 0 || decodes > 0)) break;
    const Tok restored = ptg > pr ? pdone : pdone + gen;
    if (prefill_tokens > 0 && restored == 0) {
      if (I.free_total < I.block) break;
      if (held == 0 && !alloc_block(I, id)) {
        if (!I.error) set_error(I, ERR_FIRST_BLOCK, id, 0);
        return;
      }
    } else {
      const Tok to_hold = prefill_tokens > 0 ? restored + prefill_tokens : restored + 1;
      const Tok need = block_round(to_hold, I.block) - held;
      if (need > I.free_total) break;
      for (Tok granted = 0; granted < need; granted += I.block) {
        if (!alloc_block(I, id)) {
          if (!I.error) set_error(I, ERR_ADMIT_BLOCK, id, 0);
          return;
        }
      }
    }
    wait_remove(I, id);
    LANE0(I.allowance[id] = I.true_rl[id]);
    if (restored > (Tok)I.written[id]) swap_in(I, id, restored);
    if (prefill_tokens == 0) {
      resume_decode(I, id);
    } else if (dsp < 0.0) {
      dispatch_common(I, id, prefill_tokens);
      prompts += prefill_tokens;
    } else {
      resume_prefill(I, id, prefill_tokens);
      prompts += prefill_tokens;
    }
  }
  claim_prefill_blocks(I);
  if (I.error) return;
  // prefill-only or decode-only iterations, never mixed (engine.hpp:538-542)
  LANE0(I.decode_pause = I.n_ptiter > 0 ? 1 : 0);
}

// form_sarathi (engine.hpp:565-628): chunked prefills packed with decodes.
EDEVNI void form_sarathi(Inst& I) {
  grow_decode_blocks(I);
  if (I.error) return;
  Tok budget = I.tfs - (Tok)I.R;
  // ongoing prefills first, admission order, over a copy of the list
  const int32_t no = I.n_ongo;
  for (int32_t i = LANE; i < no; i += W) I.cd_ri[i] = I.ongo[i];
  WSYNC();
  for (int32_t k = 0; k < no; ++k) {
    if (budget <= 0) break;
    const int32_t id = I.cd_ri[k];
    if (I.state[id] != ST_RUNNING) continue;
    const Tok pdone = I.prefill_done[id];
    const Tok chunk = tmin(tmin(I.chunk, (Tok)I.ptarget[id] - pdone), budget);
    if (chunk <= 0) continue;
    if (!ensure_blocks_for(I, id, pdone + chunk)) {
      if (I.error) return;
      continue;
    }
    LANE0(I.ptiter_id[I.n_ptiter] = id; I.ptiter_tok[I.n_ptiter] = (int32_t)chunk; I.n_ptiter++);
    budget -= chunk;
  }
  // new admissions
  while (budget >= 1 && I.pt_count > 0) {
    const int32_t id = wait_front(I);
    LANE0(I.exam_count++);
    const Tok pdone = I.prefill_done[id], ptg = I.ptarget[id], pr = I.prompt[id], gen = I.generated[id];
    const Tok held = I.held[id];
    const double dsp = I.dispatch_t[id];
    const Tok prefill_left = ptg - pdone;
    if (prefill_left <= 0) {  // a swapped-out decoder resuming
      const Tok resident = pr + gen;
      const Tok need = block_round(resident + 1, I.block) - held;
      if (need > I.free_total) break;
      for (Tok g = 0; g < need; g += I.block) {
        alloc_block(I, id);
        if (I.error) return;
      }
      LANE0(I.allowance[id] = I.true_rl[id]);
      swap_in(I, id, resident);
      wait_remove(I, id);
      resume_decode(I, id);
      continue;
    }
    const Tok chunk = tmin(tmin(I.chunk, prefill_left), budget);
    const Tok restored = ptg > pr ? 0 : pdone;
    if (I.free_total < I.block && held == 0) break;
    if (held == 0 && !alloc_block(I, id)) {
      if (!I.error) set_error(I, ERR_FIRST_BLOCK, id, 0);
      return;
    }
    LANE0(I.allowance[id] = I.true_rl[id]);
    if (restored > (Tok)I.written[id]) swap_in(I, id, restored);
    wait_remove(I, id);
    if (dsp < 0.0) dispatch_common(I, id, chunk); else resume_prefill(I, id, chunk);
    if (pdone + chunk < ptg) LANE0(I.ongo[I.n_ongo++] = id);
    budget -= chunk;
  }
  claim_prefill_blocks(I);
}

// commit_exact_epoch (engine.hpp:680-699)
EDEVNI void commit_exact_epoch(Inst& I, int32_t id) {
  const Tok pr = I.prompt[id], gen = I.generated[id], pad = padded_of(I, id);
  const Tok target = block_round(pr + gen + pad, I.block);
  const Tok held = I.held[id];
  bool ok = true;
  if (held == 0) ok = kvc_alloc_region(I, id, pr + gen + pad);
  else if (held < target) ok = kvc_alloc_region(I, id, target - held);
  if (I.error) return;
  if (!ok) { set_error(I, ERR_EXACT_ADMIT, id, 0); return; }
  if (LANE == 0) {
    const Tok wt = (Tok)I.prefill_done[id] + gen;
    const Tok cur = I.written[id];
    if (cur < wt) {
      I.written[id] = (int32_t)wt;
      I.written_total += wt - cur;
    }
    I.occupied[id] = (int32_t)wt;
    I.allowance[id] = (int32_t)(gen + pad);
    I.gen_epoch[id] = (int32_t)gen;
  }
  WSYNC();
}

// multires_select (policies.hpp:95-121) over wait_fifo_: the feasible
// candidate nearest (normalised Euclidean distance) to the free resources,
// first in queue order on ties. Level-1 tree nodes prune 32-id blocks whose
// smallest forward-size demand exceeds avail_gpu; the distance is computed
// exactly as the reference does (IEEE div/sqrt, no contraction).
EDEVNI int32_t multires_pick(const Inst& I, Tok avail_gpu, Tok avail_kvc) {
  const double gn = (double)tmax(1, I.tfs), kn = (double)tmax(1, I.capacity);
  double best = 0.0;
  int32_t best_id = -1;
  const int64_t nblk = I.tree_levels >= 2 ? I.tree_len[1] : 1;
  for (int64_t b0 = 0; b0 < nblk; b0 += W) {
    const int64_t bl = b0 + LANE;
    const bool live = bl < nblk && (I.tree_levels < 2 || tree_at(I, 1, bl) <= avail_gpu);
    unsigned m = BALLOT(live);
    while (m) {
      const int64_t blk = b0 + FFS(m);
      m &= m - 1;
      for (int j0 = 0; j0 < 32; j0 += W) {
        const int64_t id = blk * 32 + j0 + LANE;
        if (id < I.n && I.tree[id] <= avail_gpu) {
          const Tok gpu = I.tree[id];
          const Tok kvc = member_demand(I, (int32_t)id);
          if (kvc <= avail_kvc) {
            const double dg = ((double)gpu - (double)avail_gpu) / gn;
            const double dk = ((double)kvc - (double)avail_kvc) / kn;
            const double d = sqrt(dg * dg + dk * dk);
            if (best_id < 0 || d < best) {
              best = d;
              best_id = (int32_t)id;
            }
          }
        }
      }
    }
  }
  // (distance, id) minimum across lanes: each lane kept its first minimum
  for (int o = W / 2; o > 0; o >>= 1) {
    const double ob = shfl_xor(best, o);
    const int32_t oi = shfl_xor(best_id, o);
    const bool take = oi >= 0 && (best_id < 0 || ob < best || (ob == best && oi < best_id));
    if (take) {
      best = ob;
      best_id = oi;
    }
  }
  return best_id;
}

// form_multires (engine.hpp:658-677)
EDEVNI void form_multires(Inst& I) {
  Tok prompts = 0;
  for (;;) {
    const Tok avail_gpu = I.tfs - (Tok)I.R - prompts;
    if (avail_gpu <= 0) break;
    LANE0(I.exam_count += I.pt_count);  // one examination per waiting candidate
    const int32_t id = multires_pick(I, avail_gpu, I.free_total);
    if (id < 0) break;
    wait_remove(I, id);
    commit_exact_epoch(I, id);
    if (I.error) return;
    if (I.generated[id] > 0) {
      resume_decode(I, id);
    } else {
      dispatch_common(I, id, I.prompt[id]);
      prompts += I.prompt[id];
    }
  }
}

// form_sync_coupled (engine.hpp:704-726): same-RL groups admitted whole at
// batch boundaries, no per-iteration PT top-up.
EDEVNI void form_sync_coupled(Inst& I) {
  if (I.R == 0 && I.n_ptiter == 0) LANE0(I.admission_open = 1);
  if (!I.admission_open) return;
  int32_t nsel = 0;
  const int32_t nselg = select_gt(I, &nsel);
  if (I.error) return;
  for (int32_t i = 0; i < nsel; ++i) {
    const int32_t id = I.sel_ids[i];
    commit_exact_epoch(I, id);
    if (I.error) return;
    if (I.generated[id] > 0 || I.prefill_done[id] >= I.prompt[id]) resume_decode(I, id);
    else dispatch_common(I, id, I.prompt[id]);
  }
  if (nselg > 0) LANE0(I.admission_open = 0);
}

// form_batch (engine.hpp:249-258) for the baseline policies.
EDEVNI void form_baseline(Inst& I) {
  switch (I.policy) {
    case ECONO_POLICY_ORCA: form_orca(I); break;
    case ECONO_POLICY_VLLM: form_vllm(I); break;
    case ECONO_POLICY_SARATHI: form_sarathi(I); break;
    case ECONO_POLICY_MULTIRES: form_multires(I); break;
    default: form_sync_coupled(I); break;
  }
}
