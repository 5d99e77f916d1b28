"""K1 (device metadata builder) vs the oracle: bit-exact masks, grouping, tiles."""

import numpy as np
import pytest

import helpers
from oracle import preft_oracle as O
from paper_2605_14217_b200 import _lib
from paper_2605_14217_b200.errors import BatchError, InfeasibleBatchError

pytestmark = pytest.mark.gpu


def _flags(is_decode, all_pos):
    return (np.asarray(is_decode, dtype=np.int32) * _lib.ENTRY_DECODE
            | np.asarray(all_pos, dtype=np.int32) * _lib.ENTRY_ALL_POSITIONS).astype(np.int32)


def _check_meta(meta, qsl, slots, flags, tile_tokens, split):
    dec = (flags & _lib.ENTRY_DECODE) != 0
    allp = (flags & _lib.ENTRY_ALL_POSITIONS) != 0
    mask = O.position_mask(qsl, slots, dec, allp)
    assert np.array_equal(meta.mask_host(), mask)
    tokens, segs, tiles, offs, nsplit = O.group_by_slot(qsl, slots, dec, allp, tile_tokens, split)
    c = meta.counters_host()
    assert c[_lib.CTR_SEL_TOKENS] == len(tokens)
    assert c[_lib.CTR_SEGMENTS] == len(segs)
    assert c[_lib.CTR_TILES] == len(tiles)
    assert c[_lib.CTR_SPLIT] == nsplit
    assert c[_lib.CTR_E] == len(slots) and c[_lib.CTR_T] == qsl[-1]
    assert np.array_equal(meta.tokens_host(), tokens)
    assert np.array_equal(meta.segments_host(), segs)
    assert np.array_equal(meta.tiles_host(), tiles)
    assert np.array_equal(meta.entry_offset_host(), offs)
    chunks, units = O.chunk_units(qsl, slots, dec, allp, _lib.CHUNK_ROWS, _lib.UNIT_CHUNKS)
    assert c[_lib.CTR_CHUNKS] == len(chunks) and c[_lib.CTR_UNITS] == len(units)
    assert np.array_equal(meta.chunks_host(), chunks)
    assert np.array_equal(meta.units_host(), units)
    # LoRA-class units (slot < split) lead the unit list; their count
    u_slot = np.asarray(units).reshape(-1, 4)[:, 0]
    n_lora = int(c[_lib.CTR_LORA_UNITS])
    assert n_lora == int(np.sum(u_slot < split))
    assert (u_slot[:n_lora] < split).all() and (u_slot[n_lora:] >= split).all()
    u_nch = np.asarray(units).reshape(-1, 4)[:, 2]
    assert int(c[_lib.CTR_LORA_CHUNKS]) == int(u_nch[:n_lora].sum())
    # the LoRA units' size order K1 appends (PREFT_META_UNIT_ORDER): 4 chunks first, then
    # 3, 2, 1, unit order within a size — a stable sort by decreasing chunk count
    order = meta.unit_order_host()
    assert np.array_equal(order, np.argsort(-u_nch[:n_lora], kind="stable"))


def test_masks_and_grouping_on_golden_batches(cuda_device):
    from paper_2605_14217_b200.meta import BatchMeta

    meta = BatchMeta(64, 20000, tile_tokens=4, device=cuda_device)
    for b in helpers.mask_batches():
        qsl = b["qsl"].astype(np.int32)
        slots = b["adapter"].astype(np.int32)
        flags = _flags(b["is_decode"], b["all_pos"])
        meta.build_arrays(qsl, slots, flags)
        # the reference's PositionMask, bit for bit (model.py:305-319)
        assert np.array_equal(meta.mask_host(), b["mask"])
        _check_meta(meta, qsl, slots, flags, 4, _lib.SLOT_SPLIT_ALL_LORA)


@pytest.mark.parametrize("E,max_len,tile", [(1, 1, 1), (7, 3, 16), (300, 64, 16), (4096, 40, 16), (2000, 900, 128)])
def test_random_batches_and_split(cuda_device, E, max_len, tile):
    from paper_2605_14217_b200.meta import BatchMeta

    rng = np.random.default_rng(E * 31 + max_len)
    lens = rng.integers(1, max_len + 1, size=E)
    dec = rng.random(E) < 0.3
    lens[dec] = 1
    qsl = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    slots = rng.integers(-1, 700, size=E).astype(np.int32)
    flags = _flags(dec, rng.random(E) < 0.3)
    meta = BatchMeta(max(E, 1), int(qsl[-1]), tile_tokens=tile, device=cuda_device)
    for split in (_lib.SLOT_SPLIT_ALL_LORA, 0, 350):
        meta.set_slot_split(split)
        meta.build_arrays(qsl, slots, flags)
        _check_meta(meta, qsl, slots, flags, tile, split)


def test_all_decode_prefill_only_selects_nothing(cuda_device):
    from paper_2605_14217_b200.meta import BatchMeta

    meta = BatchMeta(8, 64, device=cuda_device)
    qsl = np.arange(6, dtype=np.int32)
    meta.build_arrays(qsl, np.arange(5, dtype=np.int32), np.full(5, _lib.ENTRY_DECODE, dtype=np.int32))
    assert not meta.mask_host().any()
    assert meta.selected_tokens() == 0
    assert meta.tiles_host().shape == (0, 4)


def test_device_rejects_malformed_offsets(cuda_device):
    from paper_2605_14217_b200.meta import BatchMeta

    meta = BatchMeta(8, 64, device=cuda_device)
    bad = (np.array([0, 3, 3, 5], dtype=np.int32), np.zeros(3, np.int32), np.zeros(3, np.int32))
    with pytest.raises(BatchError):  # the host check (default) stops it before K1
        meta.build_arrays(*bad)
    meta.build_arrays(*bad, validate=False)  # the device check: K1's error bits
    with pytest.raises(BatchError):
        meta.check_errors()
    with pytest.raises(InfeasibleBatchError):
        meta.build_arrays(np.array([0, 100], dtype=np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32))


def test_compute_position_mask_dropin_matches_reference(cuda_device):
    from paper_2605_14217_b200 import Phase, PositionSchedule, SeqEntry, compute_position_mask, make_batch

    for b in helpers.mask_batches()[:150]:
        entries = []
        for i in range(len(b["adapter"])):
            n = int(b["qsl"][i + 1] - b["qsl"][i])
            aid = int(b["adapter"][i])
            entries.append(
                SeqEntry(i, tuple(range(n)), int(b["prompt_len"][i]),
                         Phase.DECODE if b["is_decode"][i] else Phase.PREFILL,
                         None if aid < 0 else aid,
                         None if aid < 0 else (PositionSchedule.ALL_POSITIONS if b["all_pos"][i]
                                               else PositionSchedule.PREFILL_ONLY))
            )
        m = compute_position_mask(make_batch(entries))
        assert np.array_equal(m.values, b["mask"])
        assert m.uniform is b["uniform"]
