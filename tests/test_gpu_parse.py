"""Loading on the device (csrc/parse.cu, csrc/parse_tok.cuh) against the
reference's own parse_network / from_chars (oracle/_ref, io.cpp:83-175,
network.cpp:151-216): same networks, same weights bit for bit, same first
failing line and the same ParseError / ValidationError messages."""
from __future__ import annotations

import random
import struct
from decimal import Decimal, getcontext

import numpy as np
import pytest

import paper_2005_04347_b200 as A
from paper_2005_04347_b200 import _lib

pytestmark = pytest.mark.gpu


def dev_weights(tokens):
    import ctypes as C
    dev = A.Device.get(0)
    enc = [t.encode() if isinstance(t, str) else t for t in tokens]
    off = np.zeros(len(enc) + 1, np.uint64)
    off[1:] = np.cumsum([len(t) for t in enc])
    out = np.zeros(len(enc), np.float32)
    st = np.zeros(len(enc), np.uint8)
    dev.check(dev.lib.asnn_dev_parse_weights(dev.h, b"".join(enc), _lib.ptr(off, C.c_uint64), len(enc),
                                             _lib.ptr(out, C.c_float), _lib.ptr(st, C.c_uint8)))
    return out, st


def f32_from_bits(b):
    return struct.unpack("<f", struct.pack("<I", b))[0]


def weight_tokens(n, seed):
    rng = random.Random(seed)
    npr = np.random.default_rng(seed)
    toks = []
    # shortest round-trip forms (what serialize_network writes) and fixed formats
    bits = npr.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    vals = bits.view(np.float32)
    for v in vals[:n // 2]:
        if np.isfinite(v):
            toks.append(np.format_float_positional(v) if rng.random() < 0.5 else repr(float(v)))
    for v in npr.uniform(-1, 1, n // 4).astype(np.float32):
        toks.append(rng.choice(["%.9g", "%.17g", "%e", "%.3e", "%.12f", "%g"]) % float(v))
    # random digit strings: long mantissas, leading zeros, exponents
    for _ in range(n // 4):
        nd = rng.randint(1, 45)
        digits = "".join(rng.choice("0123456789") for _ in range(nd))
        if rng.random() < 0.6:
            k = rng.randint(0, nd)
            digits = digits[:k] + "." + digits[k:]
        if rng.random() < 0.7:
            digits += rng.choice("eE") + rng.choice(["", "+", "-"]) + str(rng.randint(0, 60))
        if rng.random() < 0.4:
            digits = "-" + digits
        toks.append(digits)
    return toks


def midpoint_tokens(n, seed):
    """Exact decimal expansions of float rounding midpoints, and their
    nearest neighbours one digit beyond: the ties-to-even cases."""
    getcontext().prec = 200
    rng = random.Random(seed)
    toks = []
    for _ in range(n):
        e = rng.randint(-120, 110)
        m = rng.randint(1 << 23, (1 << 24) - 1)
        mid = Decimal(2 * m + 1) * Decimal(2) ** (e - 1)
        s = format(mid, "f")
        toks.append(s)
        toks.append(s + "000001")
        toks.append(format(mid.next_minus(), "f")[:60])
    return toks


def subnormal_tokens(n, seed):
    """The float subnormal range and its edges: exact decimal expansions of
    subnormal rounding midpoints (ties to even), one digit either side,
    2^-150 (half the smallest subnormal: rounds to zero) and its neighbours,
    and subnormal values in short and long formats."""
    getcontext().prec = 250
    rng = random.Random(seed)
    toks = []
    half = Decimal(2) ** -150
    toks += [format(half, "f"), format(half, "f") + "1", format(half.next_minus(), "f")[:80],
             format(3 * half, "f"), format(3 * half, "e"), "1.4e-45", "7.0064923216240854e-46",
             format(Decimal((1 << 24) - 1) * half, "f")]  # largest subnormal / smallest normal midpoint
    for _ in range(n):
        m = rng.randint(0, (1 << 23) - 1)
        mid = Decimal(2 * m + 1) * half
        s = format(mid, "f")
        toks += [s, s + "000001", format(mid.next_minus(), "f")[:70], format(mid, "e")]
        v = struct.unpack("<f", struct.pack("<I", rng.randint(1, (1 << 23) - 1)))[0]
        toks += ["%.9g" % v, "%.3e" % v, "%.25e" % v, repr(v)]
    return toks


EDGE_TOKENS = ["1e39", "3.5e38", "3.4028235e38", "3.4028236e38", "3.40282357e38", "3.4028234664e38",
               "3.40282346638528859811704183484516925440e+38", "3.40282356779733661637539395458142568448e38",
               "1e-45", "1e-46", "7e-46", "7.1e-46", "1.4e-45", "0.7e-45", "-0", "0", "0.0", "-0.0e12",
               "inf", "-inf", "Infinity", "INF", "infin", "infinityx", "nan", "nan(123)", "NaN", "nan()",
               "nan(x_1)", "-nan", "nan(", "nan(1", ".5", "5.", ".", "-", "1e", "1e+", "0x10", "1,5", "00012",
               "1E5", "+1", "1e-38", "1.17549435e-38", "1.1754942e-38", "1e-40", "123456789012345678901234567890",
               "1.00000005960464477539062500000000000001", "1.000000059604644775390625", "0e999999",
               "1e-999999", "-1e-999999", "4294967296", "16777217", "16777216.5", "9007199254740993",
               "0.1", "0.2", "0.3", "-1", "1", "0.77743685", "-0.32799882", "1e10", "1e-10", "1e11",
               "12345678e-20", "9999999999999999999", "99999999999999999999", "1" + "0" * 60, "0." + "0" * 50 + "1"]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_weight_tokens_match_from_chars(ref, seed):
    toks = EDGE_TOKENS + weight_tokens(60000, seed) + midpoint_tokens(3000, seed) + subnormal_tokens(1500, seed)
    want, wst = ref.from_chars_f32(toks)
    got, gst = dev_weights(toks)
    # every token is decided on the device (status 0 / 1), none by the host
    assert set(np.unique(gst)) <= {0, 1}
    ok = gst == 0
    assert np.array_equal(ok, wst == 0), [t for t, a, b in zip(toks, ok, wst == 0) if a != b][:10]
    same = got.view(np.uint32) == want.view(np.uint32)
    nan = np.isnan(got) & np.isnan(want)
    bad = ok & ~(same | nan)
    assert not bad.any(), [(toks[i], got[i], want[i]) for i in np.flatnonzero(bad)[:10]]
    # the shortest round-trip forms serialize_network writes
    vals = np.random.default_rng(seed).uniform(-1, 1, 20000).astype(np.float32)
    canon = [np.format_float_positional(v, unique=True) for v in vals] + \
            [np.format_float_scientific(v, unique=True) for v in vals[:5000] * np.float32(1e-20)]
    got, gst = dev_weights(canon)
    assert not gst.any()
    assert np.array_equal(got.view(np.uint32), np.concatenate([vals, vals[:5000] * np.float32(1e-20)]).view(np.uint32))


def ref_arrays(ref, text):
    rn, err = ref.parse(text)
    return (rn.arrays(), None) if rn else (None, err)


def dev_parse(text):
    try:
        net = A.parse_network(text)
        return dict(nodes=net.nodes, inputs=net.inputs, outputs=net.outputs, source=net.source,
                    target=net.target, weight=net.weight), None
    except A.ParseError as e:
        return None, (1, e.line, str(e))
    except A.ValidationError as e:
        return None, (2, 0, str(e))


def same(ref, text):
    want, werr = ref_arrays(ref, text)
    got, gerr = dev_parse(text)
    if werr is not None:
        assert gerr is not None, (text[:200], werr)
        assert gerr[0] == werr[0] and gerr[2] == werr[2], (gerr, werr)
        if werr[0] == 1:
            assert gerr[1] == werr[1]
        return
    assert gerr is None, (gerr, text[:300])
    for k in ("nodes", "inputs", "outputs", "source", "target"):
        assert np.array_equal(got[k], want[k]), k
    assert np.array_equal(got["weight"].view(np.uint32), want["weight"].view(np.uint32))


@pytest.mark.parametrize("seed", range(6))
def test_serialized_networks_round_trip(ref, seed):
    rng = A.SplitMix64(700 + seed)
    net = ref.generate(A.random_spec(rng, 3000, 30000))
    text = ref.serialize(net)
    same(ref, text)


MALFORMED = [
    b"", b"\n", b"# only a comment\n", b"asnn 1\n", b"asnn 1\ninputs 0\n", b"asnn 2\ninputs 0\noutputs 1\n",
    b"asnn\ninputs 0\noutputs 1\n", b"asnn 1 extra\ninputs 0\noutputs 1\n", b"nets 1\n",
    b"asnn 1\noutputs 1\n", b"asnn 1\ninputs 0\nedge 0 1 0.5\n", b"asnn 1\ninputs 0 x\noutputs 1\n",
    b"asnn 1\ninputs 0\noutputs 1 -2\n", b"asnn 1\ninputs 0\noutputs 1\nedge 0 1\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5 9\n", b"asnn 1\ninputs 0\noutputs 1\nedge a 1 0.5\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 b 0.5\n", b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 w\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 1e99\n", b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 1e-99\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 1 1 0.5\n", b"asnn 1\ninputs 0\noutputs 1\nedge 007 7 0.5\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5\nedge 0 1 0.25\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5\nedge 00 01 0.25\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5\nbogus 3\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5\ninputs 2\n",
    b"asnn 1\r\ninputs 0\r\noutputs 1\r\nedge 0 1 0.5\r\n",
    b"  # lead\n\nasnn\t1\n\tinputs  0   2\n# c\noutputs 1\n\nedge 0 1 0.5\n  edge\t2 1 -0.25  \n#end",
    b"asnn 1\ninputs 4294967295\noutputs 0\nedge 4294967295 0 1\n",
    b"asnn 1\ninputs 4294967296\noutputs 0\n", b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 nan\nedge 1 2 -inf\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 1.00000005960464477539062500000000000001\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 1e-40\nedge 1 1 1e-41\n",
    b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 0.5\n#x\nedge 0 1 0.5",
]

INVALID = [
    b"asnn 1\ninputs\noutputs 1\nedge 0 1 0.5\n",
    b"asnn 1\ninputs 0\noutputs\nedge 0 1 0.5\n",
    b"asnn 1\ninputs 0 0 2 0\noutputs 1 1\nedge 0 1 0.5\nedge 2 1 0.5\n",
    b"asnn 1\ninputs 0 1\noutputs 1 2\nedge 0 2 0.5\n",
    b"asnn 1\ninputs 0 1\noutputs 2\nedge 0 1 0.5\nedge 1 2 0.5\nedge 2 0 0.1\n",
    b"asnn 1\ninputs 0\noutputs 3\nedge 0 1 1\nedge 1 2 1\nedge 2 1 1\nedge 2 3 1\n",
    b"asnn 1\ninputs 0\noutputs 5\nedge 0 5 1\nedge 7 8 1\nedge 8 9 1\nedge 9 7 1\nedge 3 4 1\nedge 4 3 1\n",
]


@pytest.mark.parametrize("i", range(len(MALFORMED)))
def test_malformed_texts(ref, i):
    same(ref, MALFORMED[i])


@pytest.mark.parametrize("i", range(len(INVALID)))
def test_validation_messages(ref, i):
    same(ref, INVALID[i])


def test_mutated_lines(ref):
    """Single-line damage anywhere in a real file: the device names the same
    first failing line and message as the sequential reference parser."""
    rng = random.Random(17)
    net = ref.generate(A.random_spec(A.SplitMix64(5), 400, 3000))
    lines = ref.serialize(net).split(b"\n")
    for _ in range(60):
        ls = list(lines)
        k = rng.randrange(len(ls))
        op = rng.randrange(5)
        if op == 0:
            ls[k] = b"edge 1 2"
        elif op == 1:
            ls.insert(k, ls[rng.randrange(3, len(ls) - 1)])   # a duplicate (or a second header...)
        elif op == 2:
            ls[k] = ls[k].replace(b" ", b"  ", 1) + b" # tail"
        elif op == 3:
            ls[k] = b"# " + ls[k]
        else:
            ls[k] = ls[k][:-1]
        same(ref, b"\n".join(ls))


def test_read_network_file(ref, tmp_path):
    net = ref.generate(A.random_spec(A.SplitMix64(8), 500, 4000))
    p = tmp_path / "net.asnn"
    p.write_bytes(ref.serialize(net))
    got = A.read_network(p)
    want = net.arrays()
    assert np.array_equal(got.nodes, want["nodes"])
    assert np.array_equal(got.weight.view(np.uint32), want["weight"].view(np.uint32))
    with pytest.raises(A.IoError):
        A.read_network(tmp_path / "missing.asnn")


def test_parse_then_activate(ref, oracle):
    """load -> levels -> activate: the parsed network goes straight through
    the device path and matches the oracle bit for bit."""
    net0 = ref.generate(A.random_spec(A.SplitMix64(31), 2000, 20000))
    net = A.parse_network(ref.serialize(net0))
    d = oracle.layout(net)
    X = np.random.default_rng(2).uniform(-2, 2, (64, len(net.inputs))).astype(np.float32)
    out, st = A.DeviceLayout.from_network(net).activate(X, state=True)
    assert np.array_equal(st.view(np.uint32), oracle.eval_batch(d, X).view(np.uint32))


def test_load_layout_on_device(ref, oracle):
    """asnn_dev_load_layout: text -> resident layout without a host round
    trip; the same layout (bitwise) and activations as parse + build."""
    net0 = ref.generate(A.random_spec(A.SplitMix64(77), 3000, 30000))
    text = ref.serialize(net0)
    dl = A.DeviceLayout.from_text(text)
    net = A.parse_network(text)
    d = oracle.layout(net)
    lay = dl.download()
    for k in ("layer_offsets", "node_ids", "row_ptr", "in_nodes"):
        assert np.array_equal(getattr(lay, k), d[k]), k
    assert np.array_equal(lay.in_weights.view(np.uint32), d["in_weights"].view(np.uint32))
    X = np.random.default_rng(1).uniform(-2, 2, (64, len(net.inputs))).astype(np.float32)
    _, st = dl.activate(X, state=True)
    assert np.array_equal(st.view(np.uint32), oracle.eval_batch(d, X).view(np.uint32))
    with pytest.raises(A.ParseError):
        A.DeviceLayout.from_text(b"asnn 1\ninputs 0\noutputs 1\nedge 0 1 x\n")
    with pytest.raises(A.ValidationError):
        A.DeviceLayout.from_text(b"asnn 1\ninputs 0\noutputs 2\nedge 0 1 1\nedge 1 2 1\nedge 2 1 1\n")


@pytest.mark.slow
def test_large_text_staged_transfers(ref):
    """Config 2's network as text (~139 MB, 5M edges): the text goes up and
    the parsed arrays (20 MB each) come back through the chunked pinned
    staging of engine.cu (upload_host / download_host, 8 MB chunks, both
    buffers and a ragged last chunk) -- same network, weights bit for bit."""
    net = A.generate_mlp(200, 500, 0.1, 2)
    text = ref.serialize(ref.network(net))
    assert len(text) > 64 << 20
    got = A.parse_network(text)
    rn, err = ref.parse(text)
    assert err is None
    want = rn.arrays()
    for k in ("nodes", "inputs", "outputs", "source", "target"):
        assert np.array_equal(getattr(got, k), want[k]), k
    assert np.array_equal(got.weight.view(np.uint32), want["weight"].view(np.uint32))
