"""Decode stage on the GPU: the paged GQA decode
attention kernel against an fp32 torch restatement, and the decode loop of
the decoder (first tokens from prefill, then one token per step through the
paged arena) against the fp32 oracle's full recompute."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref_decode(q, K, V, bt, bt_off, kv_len, hq, hkv, hd, scale):
    out = []
    G = hq // hkv
    for r in range(q.shape[0]):
        slots = bt[bt_off[r]:bt_off[r] + kv_len[r]].long()
        k = K[slots].float().view(-1, hkv, hd)
        v = V[slots].float().view(-1, hkv, hd)
        qq = q[r].float().view(hkv, G, hd)
        s = torch.einsum("hgd,thd->hgt", qq, k) * scale
        p = torch.softmax(s, -1)
        out.append(torch.einsum("hgt,thd->hgd", p, v).reshape(-1))
    return torch.stack(out)


@pytest.mark.parametrize("hq,hkv,hd", [(28, 4, 128), (32, 32, 128), (4, 2, 64), (64, 8, 128),
                                       (16, 1, 64)])
@pytest.mark.parametrize("lens", [[1, 31, 32, 33, 200], [7000, 5, 4097], [1] * 64,
                                  [300] * 3 + [12000],
                                  # mixed lengths: splits sized per request (one long row
                                  # among short ones), and > 512 requests (two launches)
                                  [15000] + [17 * i % 900 + 1 for i in range(63)],
                                  [(37 * i) % 700 + 1 for i in range(600)]])
def test_decode_attention(hq, hkv, hd, lens):
    from paper_2507_10069_b200 import ops
    g = torch.Generator(device="cuda").manual_seed(sum(lens) + hq)
    n_slots = sum(lens) + 500
    K = torch.randn(n_slots, hkv * hd, device="cuda", generator=g).bfloat16()
    V = torch.randn(n_slots, hkv * hd, device="cuda", generator=g).bfloat16()
    perm = torch.randperm(n_slots, device="cuda", generator=g).to(torch.int32)
    bt = perm[:sum(lens)].contiguous()                    # scattered token slots
    off = [0]
    for x in lens:
        off.append(off[-1] + x)
    bt_off = torch.tensor(off, dtype=torch.int64, device="cuda")
    kv_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    q = (torch.randn(len(lens), hq * hd, device="cuda", generator=g) * 2).bfloat16()
    out = ops.decode_attention(q, K, V, bt, bt_off, kv_len, hkv, hd, max(lens))
    torch.cuda.synchronize()
    ref = _ref_decode(q, K, V, bt.cpu().cuda(), off, lens, hq, hkv, hd, hd ** -0.5)
    assert torch.isfinite(out.float()).all()
    err = (out.float() - ref).norm() / ref.norm()
    assert err.item() < 1e-2, err.item()
    # per-row check too (a wrong split merge would hide in the global norm)
    row_err = (out.float() - ref).norm(dim=1) / ref.norm(dim=1)
    assert row_err.max().item() < 2e-2


def test_decode_attention_strided_q_and_kv_plane():
    """q rows with a pitch (a view into a fused buffer) and a K/V plane that is
    one layer of a [L, 2, slots, kv_dim] arena."""
    from paper_2507_10069_b200 import ops
    hq, hkv, hd, L = 8, 2, 128, 3
    lens = [129, 64, 1]
    g = torch.Generator(device="cuda").manual_seed(5)
    arena = torch.randn(L, 2, 400, hkv * hd, device="cuda", generator=g).bfloat16()
    qbuf = torch.randn(len(lens), hq * hd + 64, device="cuda", generator=g).bfloat16()
    q = qbuf[:, :hq * hd]
    bt = torch.arange(sum(lens), dtype=torch.int32, device="cuda") * 2
    off = [0, 129, 193, 194]
    bt_off = torch.tensor(off, dtype=torch.int64, device="cuda")
    kv_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = ops.decode_attention(q, arena[1, 0], arena[1, 1], bt, bt_off, kv_len, hkv, hd,
                               max(lens))
    ref = _ref_decode(q, arena[1, 0], arena[1, 1], bt, off, lens, hq, hkv, hd, hd ** -0.5)
    err = (out.float() - ref).norm() / ref.norm()
    assert err.item() < 1e-2


def _shape(name, dec_layers=None):
    import dataclasses
    from paper_2507_10069_b200 import shapes
    s = shapes.SHAPES[name]
    s = dataclasses.replace(s, vision=dataclasses.replace(s.vision, layers=1))
    if dec_layers is not None:
        s = dataclasses.replace(s, decoder=dataclasses.replace(s.decoder, layers=dec_layers))
    return s


def _oracle_logits(hp, req, gen):
    """fp32 full recompute of prompt + generated tokens (oracle/model_ref.py),
    inputs = the product's bf16 embedding rows / image slabs."""
    from oracle import model_ref
    from paper_2507_10069_b200.keys import TAG_IMG, request_keys
    keys, w = request_keys(hp.codec, req)
    emb = hp.Wd["embed"]
    rows = []
    for k, ww in zip(keys, w):
        if int(k) >> 62 == TAG_IMG:
            rows.append(hp.slabs[hp.codec.symbol(int(k))[1]].float())
        else:
            rows.append(emb[int(k) % hp.shape.decoder.vocab].float()[None])
    rows += [emb[g].float()[None] for g in gen]
    pos3 = None
    if hp.shape.decoder.mrope_section:
        syms = [("img", int(ww)) if int(k) >> 62 == TAG_IMG else ("txt", 1)
                for k, ww in zip(keys, w)] + [("txt", 1)] * len(gen)
        pos3 = model_ref.mrope_positions_ref(syms)
    return model_ref.decoder_ref(hp.shape, hp.Wd, torch.cat(rows, 0), pos3=pos3)[3]


@pytest.mark.parametrize("graphs,nan_mem", [(False, False), (True, False), (True, True)])
@pytest.mark.parametrize("name,layers", [("tiny", None), ("qwen-7b", 2), ("llava-7b", 2)])
def test_decode_matches_full_recompute(name, layers, graphs, nan_mem):
    """Prefill, then continuous-batching decode through the paged arena:
    every step's logits of every request equal the fp32 oracle's full
    recompute of its prompt + the tokens generated so far (rtol 2e-2);
    requests retire after output_len tokens and free their slots."""
    from paper_2507_10069_b200.decode import DecodeSession
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import ImageInput, Request
    shape = _shape(name, layers)
    hp = HotPath(shape, budget_tokens=20000)
    tok = 576 if name == "llava-7b" else 64
    X = ImageInput("4" * 32, tok, (0, 0))
    reqs = [Request(0, 0.0, "multimodal", 40, (X,), 6, prefix_id=3, prefix_len=8),
            Request(1, 0.0, "text", 17, (), 3),
            Request(2, 0.0, "multimodal", 9, (X,), 1),
            Request(3, 0.0, "text", 120, (), 9)]
    hp.encode([X])
    if nan_mem:   # buffers allocated from here on start as NaN, not as fresh zeros
        junk = torch.full((1 << 31,), float("nan"), device="cuda", dtype=torch.bfloat16)
        del junk
    res = hp.prefill(reqs, [0] * len(reqs))
    n_slots = sum(r.total_input_len + r.output_len for r in reqs) + 64
    sess = DecodeSession(hp, n_slots, graphs=graphs)
    sess.admit(res.kv, reqs, res.next_ids)
    first = res.next_ids.cpu().tolist()
    gen = {r.id: [first[i]] for i, r in enumerate(reqs)}
    by_id = {r.id: r for r in reqs}
    assert [a.rid for a in sess.active] == [0, 1, 3]     # request 2 wants one token only
    while sess.active:
        rids = [a.rid for a in sess.active]
        ids, logits = sess.step(return_logits=True)
        ids = ids.cpu().tolist()
        for i, rid in enumerate(rids):
            ref = _oracle_logits(hp, by_id[rid], gen[rid])
            err = ((logits[i].float() - ref).norm() / ref.norm()).item()
            assert err < 2e-2, (rid, len(gen[rid]), err)
            gen[rid].append(ids[i])
    for r in reqs:
        assert len(gen[r.id]) == r.output_len
    assert sess.arena.free_slots == n_slots
    assert sess.generated == sum(r.output_len - 1 for r in reqs)


def test_decode_graph_session_joins_and_retires():
    """CUDA-graph decode with requests joining mid-stream and retiring at
    different steps (bucket changes 1 -> 2 -> 4 -> 2): tokens equal the eager
    session's step by step."""
    from paper_2507_10069_b200.decode import DecodeSession
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import Request
    hp = HotPath(_shape("tiny"), budget_tokens=20000)
    reqs = [Request(i, 0.0, "text", 20 + 7 * i, (), 3 + 4 * (i % 3)) for i in range(5)]
    out = {}
    for graphs in (False, True):
        sess = DecodeSession(hp, 4096, graphs=graphs)
        toks = {r.id: [] for r in reqs}
        plan = {0: [0], 2: [1, 2], 5: [3, 4]}            # step -> requests admitted
        step = 0
        while step < 40 and (sess.active or any(k >= step for k in plan)):
            if step in plan:
                batch = [reqs[i] for i in plan[step]]
                res = hp.prefill(batch, [0] * len(batch))
                sess.admit(res.kv, batch, res.next_ids)
                hp.release_batch_kv()
            rids = [a.rid for a in sess.active]
            o = sess.step()
            if o is not None:
                for rid, t in zip(rids, o.cpu().tolist()):
                    toks[rid].append(t)
            step += 1
        out[graphs] = toks
        assert not sess.active and sess.arena.free_slots == 4096
    assert out[True] == out[False]


@pytest.mark.parametrize("graphs", [False, True])
@pytest.mark.parametrize("name,layers", [("tiny-x", None), ("llama-11b-v", 5)])
def test_cross_model_decode_matches_full_recompute(name, layers, graphs):
    """Decode of the cross-attention model (Llama-3.2-Vision): text K/V in
    the self planes, the images' cross K/V read through their own block
    tables; a text-only request in the same batch skips the cross layers
    (masked MLP).  Logits vs the fp32 oracle's full recompute each step."""
    import dataclasses
    from oracle import model_ref
    from paper_2507_10069_b200 import shapes
    from paper_2507_10069_b200.decode import DecodeSession
    from paper_2507_10069_b200.keys import TAG_IMG, request_keys
    from paper_2507_10069_b200.pipeline import HotPath
    from paper_2507_10069_b200.workload import ImageInput, Request
    s = shapes.SHAPES[name]
    s = dataclasses.replace(s, vision=dataclasses.replace(s.vision, layers=1))
    if layers is not None:
        s = dataclasses.replace(s, decoder=dataclasses.replace(s.decoder, layers=layers))
    hp = HotPath(s, budget_tokens=20000)
    tok = 576 if name == "llama-11b-v" else 64
    X = ImageInput("8" * 32, tok, (0, 0))
    Y = ImageInput("9" * 32, tok // 2, (0, 0))
    reqs = [Request(0, 0.0, "multimodal", 30, (X,), 5, prefix_id=2, prefix_len=8),
            Request(1, 0.0, "text", 19, (), 4),
            Request(2, 0.0, "multimodal", 11, (Y, X), 6)]
    hp.encode([X, Y])
    res = hp.prefill(reqs, [0] * len(reqs))
    sess = DecodeSession(hp, sum(r.total_input_len + r.output_len for r in reqs) + 64,
                         graphs=graphs)
    sess.admit(res.kv, reqs, res.next_ids)
    hp.release_batch_kv()
    first = res.next_ids.cpu().tolist()
    gen = {r.id: [first[i]] for i, r in enumerate(reqs)}
    by_id = {r.id: r for r in reqs}
    emb = hp.Wd["embed"]

    def oracle(req, g):
        keys, w = request_keys(hp.codec, req)
        txt, img = [], []
        for k, ww in zip(keys, w):
            if int(k) >> 62 == TAG_IMG:
                img.append(hp.slabs[hp.codec.symbol(int(k))[1]].float())
            else:
                txt.append(emb[int(k) % s.decoder.vocab].float()[None])
        txt += [emb[t].float()[None] for t in g]
        return model_ref.decoder_ref(s, hp.Wd, torch.cat(txt, 0),
                                     img=torch.cat(img, 0) if img else None)[3]
    while sess.active:
        rids = [a.rid for a in sess.active]
        ids, logits = sess.step(return_logits=True)
        ids = ids.cpu().tolist()
        for i, rid in enumerate(rids):
            ref = oracle(by_id[rid], gen[rid])
            assert torch.isfinite(ref).all(), ("oracle", rid)
            assert torch.isfinite(logits[i].float()).all(), ("product", rid, len(gen[rid]))
            err = ((logits[i].float() - ref).norm() / ref.norm()).item()
            assert err < 2e-2, (rid, len(gen[rid]), err)
            gen[rid].append(ids[i])
    for r in reqs:
        assert len(gen[r.id]) == r.output_len


def test_decode_attention_zero_length_rows():
    """Padding rows of a CUDA-graph batch have kv_len 0: their output is 0 and
    they do not disturb the other rows' splits."""
    from paper_2507_10069_b200 import ops
    hq, hkv, hd = 28, 4, 128
    lens = [0, 5, 0, 3000, 0]
    g = torch.Generator(device="cuda").manual_seed(11)
    n_slots = sum(lens) + 64
    K = torch.randn(n_slots, hkv * hd, device="cuda", generator=g).bfloat16()
    V = torch.randn(n_slots, hkv * hd, device="cuda", generator=g).bfloat16()
    bt = torch.randperm(n_slots, device="cuda", generator=g)[:sum(lens)].to(torch.int32)
    off = [0]
    for x in lens:
        off.append(off[-1] + x)
    bt_off = torch.tensor(off, dtype=torch.int64, device="cuda")
    kv_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    q = torch.randn(len(lens), hq * hd, device="cuda", generator=g).bfloat16()
    out = ops.decode_attention(q, K, V, bt, bt_off, kv_len, hkv, hd, max(lens))
    live = [1, 3]
    ref = _ref_decode(q[live], K, V, bt, [off[i] for i in live], [lens[i] for i in live],
                      hq, hkv, hd, hd ** -0.5)
    assert (out[[0, 2, 4]] == 0).all()
    err = (out[live].float() - ref).norm(dim=1) / ref.norm(dim=1)
    assert err.max().item() < 2e-2
