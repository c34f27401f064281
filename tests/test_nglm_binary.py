"""NGLM binary model files (format SPEC.md:209) on CPU: the
file layout read back with `struct` field by field, the CRC-32 against zlib's,
round trips bit-identical (arrays, header info, state_of on random histories:
pins the prefix-edge map rebuilt from the flat arrays), and each corruption
rejected with its own error."""
import struct
import zlib

import numpy as np
import pytest

import paper_2505_22857_b200 as ng

NAMES = ["uni16", "bi16", "tiny3", "tri64", "five48", "ten24"]


def models(small_lms, fig1_paths, tmp_path):
    out = [("fig1", ng.load_arpa(*fig1_paths, device=-1))]
    for n in NAMES:
        f = small_lms[n]
        out.append((n, ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=-1)))
    return out


def test_file_layout_and_crc(small_lms, tmp_path):
    f = small_lms["five48"]
    m = ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=-1)
    p = str(tmp_path / "m.nglm")
    m.save(p)
    b = open(p, "rb").read()
    assert b[:4] == b"NGLM"
    version, order, V, S, A, root, bos = struct.unpack_from("<IIIIQII", b, 4)
    assert (version, order, V, S, A, root, bos) == (1, m.order, m.V, m.num_states, m.info.num_arcs, 0, m.bos_state)
    h = m.host_arrays()
    off = 36
    for name, dt, n in (("arc_tokens", "<u4", A), ("arc_weights", "<f4", A), ("arc_to_states", "<u4", A)):
        a = np.frombuffer(b, dtype=dt, count=n, offset=off)
        assert np.array_equal(a.view(np.int32), h[name].view(np.int32)), name
        off += 4 * n
    start = np.frombuffer(b, dtype="<u8", count=S, offset=off); off += 8 * S
    end = np.frombuffer(b, dtype="<u8", count=S, offset=off); off += 8 * S
    assert np.array_equal(start, h["arc_offsets"][:-1]) and np.array_equal(end, h["arc_offsets"][1:])
    for name, dt in (("boff_weights", "<f4"), ("boff_to_states", "<u4"), ("final_weights", "<f4")):
        a = np.frombuffer(b, dtype=dt, count=S, offset=off)
        assert np.array_equal(a.view(np.int32), h[name].view(np.int32)), name
        off += 4 * S
    assert off + 4 == len(b)
    assert struct.unpack_from("<I", b, off)[0] == zlib.crc32(b[:off])


def test_round_trip_bit_identical(small_lms, fig1_paths, tmp_path):
    rng = np.random.default_rng(3)
    for name, m in models(small_lms, fig1_paths, tmp_path):
        p = str(tmp_path / f"{name}.nglm")
        m.save(p)
        r = ng.load_binary(p, device=-1)
        a, b = m.host_arrays(), r.host_arrays()
        for k in a:
            assert np.array_equal(a[k].view(np.int32), b[k].view(np.int32)), (name, k)
        for k in ("order", "vocab_size", "num_states", "bos_state", "num_arcs"):
            assert getattr(m.info, k) == getattr(r.info, k), (name, k)
        if m.order >= 2:
            assert r.info.num_unk_filled == m.info.num_unk_filled
        assert r.info.num_dropped == -1
        # prefix edges rebuilt from the arrays: state_of agrees on random histories
        for _ in range(300):
            n = int(rng.integers(0, 2 * m.order + 2))
            toks = rng.integers(0, m.V, size=n).tolist()
            bos = bool(rng.integers(2))
            assert r.state_of(bos, toks) == m.state_of(bos, toks), (name, bos, toks)
        # and on histories that exist in the LM (replayed sentences)
        if name != "fig1":
            sents = [list(map(int, line.split())) for line in open(small_lms[name].heldout) if line.strip()]
            for s in sents[:30]:
                for i in range(len(s) + 1):
                    assert r.state_of(True, s[:i]) == m.state_of(True, s[:i])
        # save(load(save(m))) is byte-identical
        p2 = str(tmp_path / f"{name}_2.nglm")
        r.save(p2)
        assert open(p, "rb").read() == open(p2, "rb").read()


def test_corruptions_rejected(small_lms, tmp_path):
    f = small_lms["tri64"]
    m = ng.load_arpa(f.arpa, vocab_size=f.vocab_size, device=-1)
    p = tmp_path / "m.nglm"
    m.save(str(p))
    good = p.read_bytes()

    def expect(data, msg):
        q = tmp_path / "bad.nglm"
        q.write_bytes(data)
        with pytest.raises(ng.NgpulmError) as e:
            ng.load_binary(str(q), device=-1)
        assert msg in str(e.value) and e.value.code == ng.NGPULM_EDOMAIN

    expect(b"XGLM" + good[4:], "bad magic")
    expect(good[:4] + struct.pack("<I", 999) + good[8:], "unsupported version")
    expect(good[:20], "truncated")
    expect(good[:-10], "truncated")
    flip = bytearray(good)
    flip[100] ^= 0x40
    expect(bytes(flip), "checksum mismatch")
    with pytest.raises(ng.NgpulmError) as e:
        ng.load_binary(str(tmp_path / "missing.nglm"), device=-1)
    assert e.value.code == ng.NGPULM_EIO
