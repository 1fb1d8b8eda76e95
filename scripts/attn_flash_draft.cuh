// Draft: flash-decoding attention body with the split merge in the consumer GEMV
// prologue (x mode 2).  Correct (GPU parity green) but slower than the split+merge
// stages at s=1024 (CUDA-core scores/PV are shared-memory bound); kept for the
// tensor-core rewrite.
// Split-K decode attention (flash-decoding) for kv head g, split c.  The
// split's K/V position blocks arrive through the ring interleaved (K0 V0 K1
// V1 ...); every block updates an online softmax: scores (one (position, head)
// dot product per thread), per-head running max / sum (warp per head), then
// the P.V accumulation with the thread owning (head, dim pair) outputs in
// registers across blocks.  The last split also folds in the new token at
// position s, whose K/V row the QKV epilogue wrote before the QKV Event Tensor
// fired (read from L2 after the wait, never from the prefetched ring).  The
// unnormalised partial (m, l, o) per q head is merged by the consumer GEMV's
// prologue (x mode 2), so no separate merge stage or hop exists.
__device__ void body_attn(const StaticParams& P, const et_op& op, const SlotView& si, float* scratch, Ring& ring,
                          int ctid) {
    constexpr int kMaxOut = 4;  // (head, dim pair) outputs per thread: G * dh / 2 <= 1024
    const int warp = ctid >> 5, lane = ctid & 31;
    const int dh = op.i[0], G = op.i[1], PB = op.i[2], cap = op.i[3], NS = op.i[5];
    const long long s = P.binding[op.i[4]];
    const int g = si.coord[0], c = si.coord[1];
    const AttnSpan span = attn_span(op, c, P.binding);
    const bool last = c == NS - 1;
    const int qstride = dh + 4;          // padded rows: heads land on different banks
    const int nvec = dh / 8;             // 16-byte vectors per K/V row
    const int half = dh / 2;
    float* qs = scratch;                 // [G][dh+4]
    float* sc = qs + G * qstride;        // [G][PB] scores -> probabilities
    float* st = sc + G * PB;             // [G][4]: m, l, alpha (block rescale)
    const float* q = reinterpret_cast<const float*>(op.p[0]) + static_cast<long long>(g) * G * dh;
    if (!(P.debug & 1024))
        for (int i = ctid; i < G * dh; i += kConsumers) qs[(i / dh) * qstride + i % dh] = __ldcg(q + i);
    if (ctid < G) {
        st[ctid * 4 + 0] = -INFINITY;
        st[ctid * 4 + 1] = 0.f;
    }
    bar_sync(1, kConsumers);
    const float scale = op.f[0];
    float o0[kMaxOut], o1[kMaxOut];
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) o0[j] = o1[j] = 0.f;

    const int nblk = (span.np + PB - 1) / PB;
    for (int b = 0; b < nblk; ++b) {
        const int np = span.np - b * PB < PB ? span.np - b * PB : PB;
        const unsigned long long ck = ring.seq, cv = ring.seq + 1;
        ring.seq += 2;
        const uint8_t* kb = ring.wait(ck);
        if (!kb) return;
        // scores; each position starts its walk over the row at a different 16-byte
        // vector (bank rotation)
        for (int t = ctid; t < ((P.debug & 128) ? 0 : G * np); t += kConsumers) {
            const int h = t % G, p = t / G;
            const uint8_t* kr = kb + p * dh * 2;
            const float* qh = qs + h * qstride;
            float a0 = 0.f, a1 = 0.f;
            for (int v = 0; v < nvec; ++v) {
                const int vv = (v + p) & (nvec - 1);
                const uint4 k8 = lds128(kr + vv * 16);
                const float4 qa = *reinterpret_cast<const float4*>(qh + vv * 8);
                const float4 qb = *reinterpret_cast<const float4*>(qh + vv * 8 + 4);
                a0 = fmaf(bf16lo(k8.x), qa.x, a0);
                a1 = fmaf(bf16hi(k8.x), qa.y, a1);
                a0 = fmaf(bf16lo(k8.y), qa.z, a0);
                a1 = fmaf(bf16hi(k8.y), qa.w, a1);
                a0 = fmaf(bf16lo(k8.z), qb.x, a0);
                a1 = fmaf(bf16hi(k8.z), qb.y, a1);
                a0 = fmaf(bf16lo(k8.w), qb.z, a0);
                a1 = fmaf(bf16hi(k8.w), qb.w, a1);
            }
            sc[h * PB + p] = (a0 + a1) * scale;
        }
        bar_sync(1, kConsumers);
        if (ctid == Ring::owner(ck) * 32) ring.release(ck);
        // online softmax statistics per head (warp h)
        for (int h = warp; h < G; h += kConsumerWarps) {
            float m = -INFINITY;
            for (int p = lane; p < np; p += 32) m = fmaxf(m, sc[h * PB + p]);
            m = warp_max(m);
            const float mo = st[h * 4], mn = fmaxf(mo, m);
            float l = 0.f;
            for (int p = lane; p < np; p += 32) {
                const float e = __expf(sc[h * PB + p] - mn);
                sc[h * PB + p] = e;
                l += e;
            }
            l = warp_sum(l);
            if (lane == 0) {
                const float alpha = __expf(mo - mn);  // 0 for the first block (mo = -inf)
                st[h * 4 + 0] = mn;
                st[h * 4 + 1] = st[h * 4 + 1] * alpha + l;
                st[h * 4 + 2] = alpha;
            }
        }
        bar_sync(1, kConsumers);
        const uint8_t* vb = ring.wait(cv);
        if (!vb) return;
        const uint32_t* v2 = reinterpret_cast<const uint32_t*>(vb);
#pragma unroll
        for (int j = 0; j < kMaxOut; ++j) {
            const int idx = ctid + j * kConsumers;
            if (idx >= G * half || (P.debug & 256)) break;
            const int h = idx / half, dp = idx % half;
            const float* ph = sc + h * PB;
            const float alpha = st[h * 4 + 2];
            float a0 = o0[j] * alpha, a1 = o1[j] * alpha, a2 = 0.f, a3 = 0.f;
            int p = 0;
#pragma unroll 4
            for (; p + 2 <= np; p += 2) {
                const uint32_t va = v2[p * half + dp], vb2 = v2[(p + 1) * half + dp];
                const float wa = ph[p], wb = ph[p + 1];
                a0 = fmaf(wa, bf16lo(va), a0);
                a1 = fmaf(wa, bf16hi(va), a1);
                a2 = fmaf(wb, bf16lo(vb2), a2);
                a3 = fmaf(wb, bf16hi(vb2), a3);
            }
            if (p < np) {
                const uint32_t va = v2[p * half + dp];
                a0 = fmaf(ph[p], bf16lo(va), a0);
                a1 = fmaf(ph[p], bf16hi(va), a1);
            }
            o0[j] = a0 + a2;
            o1[j] = a1 + a3;
        }
        bar_sync(1, kConsumers);  // sc / st are reused by the next block
        if (ctid == Ring::owner(cv) * 32) ring.release(cv);
    }

    if (last) {  // the new token at position s
        const uint16_t* kn = reinterpret_cast<const uint16_t*>(op.p[1]) + (static_cast<long long>(g) * cap + s) * dh;
        for (int h = warp; h < G; h += kConsumerWarps) {
            const float* qh = qs + h * qstride;
            float dot = 0.f;
            for (int d = lane; d < dh; d += 32) dot += qh[d] * bf2f(__ldcg(kn + d));
            dot = warp_sum(dot) * scale;
            if (lane == 0) {
                const float mo = st[h * 4], mn = fmaxf(mo, dot);
                const float alpha = __expf(mo - mn), e = __expf(dot - mn);
                st[h * 4 + 0] = mn;
                st[h * 4 + 1] = st[h * 4 + 1] * alpha + e;
                st[h * 4 + 2] = alpha;
                st[h * 4 + 3] = e;
            }
        }
        bar_sync(1, kConsumers);
        const uint32_t* vn = reinterpret_cast<const uint32_t*>(op.p[2]) + (static_cast<long long>(g) * cap + s) * half;
#pragma unroll
        for (int j = 0; j < kMaxOut; ++j) {
            const int idx = ctid + j * kConsumers;
            if (idx >= G * half) break;
            const int h = idx / half, dp = idx % half;
            const uint32_t vv = __ldcg(vn + dp);
            const float alpha = st[h * 4 + 2], e = st[h * 4 + 3];
            o0[j] = fmaf(e, bf16lo(vv), o0[j] * alpha);
            o1[j] = fmaf(e, bf16hi(vv), o1[j] * alpha);
        }
    }
    // unnormalised partial of q head (g*G + h), split c: o -> p3 [q_heads][NS][dh],
    // (m, l) -> p4 [q_heads][NS]
    float* po = reinterpret_cast<float*>(op.p[3]);
    float2* pml = reinterpret_cast<float2*>(op.p[4]);
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) {
        const int idx = ctid + j * kConsumers;
        if (idx >= G * half) break;
        const int h = idx / half, dp = idx % half;
        const long long hc = (static_cast<long long>(g) * G + h) * NS + c;
        *reinterpret_cast<float2*>(po + hc * dh + 2 * dp) = make_float2(o0[j], o1[j]);
        if (dp == 0) pml[hc] = make_float2(st[h * 4], st[h * 4 + 1]);
    }
}


// body_gemv prologue, x mode 2 (merge of the flash-decoding partials):
    if (op.i[3] == 2) {
        // merge of the attention splits (x = attention output, bf16):
        //   x[h][d] = sum_c e^(m_c - M) o_c[d] / sum_c e^(m_c - M) l_c,  M = max_c m_c
        // The o partials of this thread's outputs are loaded into registers in the
        // same round trip as the split statistics.
        constexpr int kV = 4, kMaxNS = 4;
        const int NS = op.i[8], dh = op.i[9], nh = K / dh;
        const float4* po = reinterpret_cast<const float4*>(op.p[2]);  // [nh][NS][dh]
        const float2* pml = reinterpret_cast<const float2*>(op.p[3]);  // [nh][NS] (m, l)
        float* w = acc;                                                // [nh][NS] weights
        const int dh4 = dh / 4;
        for (int base = 0; base < K / 4; base += kV * kConsumers) {
            float4 ov[kV][kMaxNS];
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const int i4 = base + v * kConsumers + ctid;
                const int h = i4 / dh4, d4 = i4 - h * dh4;
#pragma unroll
                for (int cc = 0; cc < kMaxNS; ++cc)
                    if (i4 < K / 4 && cc < NS) ov[v][cc] = __ldcg(po + (static_cast<long long>(h) * NS + cc) * dh4 + d4);
            }
            if (base == 0) {
                for (int h = ctid; h < nh; h += kConsumers) {
                    float2 ml[kMaxNS];
                    float M = -INFINITY;
#pragma unroll
                    for (int cc = 0; cc < kMaxNS; ++cc)
                        if (cc < NS) {
                            ml[cc] = __ldcg(pml + h * NS + cc);
                            M = fmaxf(M, ml[cc].x);
                        }
                    float L = 0.f;
#pragma unroll
                    for (int cc = 0; cc < kMaxNS; ++cc)
                        if (cc < NS) {
                            ml[cc].x = ml[cc].x == -INFINITY ? 0.f : __expf(ml[cc].x - M);
                            L += ml[cc].x * ml[cc].y;
                        }
                    const float inv = 1.f / L;
#pragma unroll
                    for (int cc = 0; cc < kMaxNS; ++cc)
                        if (cc < NS) w[h * NS + cc] = ml[cc].x * inv;
                }
                bar_sync(1, kConsumers);
            }
#pragma unroll
            for (int v = 0; v < kV; ++v) {
                const int i4 = base + v * kConsumers + ctid;
                if (i4 >= K / 4) break;
                const int h = i4 / dh4;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int cc = 0; cc < kMaxNS; ++cc)
                    if (cc < NS) {
                        const float wt = w[h * NS + cc];
                        o.x = fmaf(wt, ov[v][cc].x, o.x);
                        o.y = fmaf(wt, ov[v][cc].y, o.y);
                        o.z = fmaf(wt, ov[v][cc].z, o.z);
                        o.w = fmaf(wt, ov[v][cc].w, o.w);
                    }
                uint2 pk;
                pk.x = static_cast<uint32_t>(f2bf(o.x)) | (static_cast<uint32_t>(f2bf(o.y)) << 16);
                pk.y = static_cast<uint32_t>(f2bf(o.z)) | (static_cast<uint32_t>(f2bf(o.w)) << 16);
                *reinterpret_cast<uint2*>(xs + i4 * 4) = pk;
            }
        }
        bar_sync(1, kConsumers);  // w (in acc) is read before acc is zeroed below
    }
