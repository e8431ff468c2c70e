"""Randomised loader parity (GPU): serialized reference-generator networks
damaged by random byte- and token-level mutations (one to three per file),
parsed by the device loader (csrc/parse.cu) and by the reference's own
parse_network (oracle/_ref, io.cpp:83-175 + validate, network.cpp:151-216).
Outcome, exception class, first failing line and message must agree; on
success the arrays must be equal bit for bit.  Runs until the time budget is
spent and prints one summary line (profiles/r1_fuzz.txt).

    python tools/fuzz_parse.py [seconds] [seed]"""
import json
import random
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2005_04347_b200 as A  # noqa: E402
from oracle.bind import Ref  # noqa: E402

TOKENS = [b"asnn", b"1", b"2", b"inputs", b"outputs", b"edge", b"#", b"-", b"+", b"0", b"00", b"4294967295",
          b"4294967296", b"1e39", b"1e-46", b"nan", b"inf", b"-0", b"0x10", b"1.5e", b".", b"e5", b"\t", b"\r",
          b" ", b"", b"0.30000001192092896", b"3.4028235e38", b"1.17549435e-38", b"7"]


def mutate(rng, text):
    lines = text.split(b"\n")
    for _ in range(rng.randint(1, 3)):
        k = rng.randrange(len(lines))
        op = rng.randrange(9)
        ln = lines[k]
        if op == 0 and ln:                       # delete a byte
            i = rng.randrange(len(ln))
            lines[k] = ln[:i] + ln[i + 1:]
        elif op == 1:                            # insert a byte
            i = rng.randrange(len(ln) + 1)
            lines[k] = ln[:i] + bytes([rng.choice(b"0123456789 -+.eE#\tx")]) + ln[i:]
        elif op == 2:                            # replace a token
            toks = ln.split(b" ")
            toks[rng.randrange(len(toks))] = rng.choice(TOKENS)
            lines[k] = b" ".join(toks)
        elif op == 3:                            # duplicate a line
            lines.insert(k, lines[rng.randrange(len(lines))])
        elif op == 4:                            # drop a line
            del lines[k]
            if not lines:
                lines = [b""]
        elif op == 5:                            # swap two lines
            j = rng.randrange(len(lines))
            lines[k], lines[j] = lines[j], lines[k]
        elif op == 6:                            # append a token
            lines[k] = ln + b" " + rng.choice(TOKENS)
        elif op == 7:                            # comment it out
            lines[k] = b"# " + ln
        else:                                    # perturb a weight's digits
            toks = ln.split(b" ")
            if len(toks) == 4 and toks[0] == b"edge":
                w = toks[3]
                i = rng.randrange(len(w)) if w else 0
                toks[3] = w[:i] + bytes([rng.choice(b"0123456789")]) + w[i + 1:]
                lines[k] = b" ".join(toks)
    return b"\n".join(lines)


def outcome_ref(ref, text):
    rn, err = ref.parse(text)
    return (rn.arrays(), None) if rn else (None, err)


def outcome_dev(text):
    try:
        net = A.parse_network(text)
        return dict(nodes=net.nodes, inputs=net.inputs, outputs=net.outputs, source=net.source,
                    target=net.target, weight=net.weight), None
    except A.ParseError as e:
        return None, (1, e.line, str(e))
    except A.ValidationError as e:
        return None, (2, 0, str(e))


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = random.Random(seed)
    sm = A.SplitMix64(seed)
    ref = Ref()
    st = {"files": 0, "parsed_ok": 0, "parse_errors": 0, "validation_errors": 0, "mismatches": 0}
    bad = []
    t_end = time.perf_counter() + budget
    while time.perf_counter() < t_end:
        net = ref.generate(A.random_spec(sm, 20, rng.choice([200, 2000, 20000])))
        base = ref.serialize(net)
        for _ in range(8):
            text = mutate(rng, base)
            want, werr = outcome_ref(ref, text)
            got, gerr = outcome_dev(text)
            st["files"] += 1
            ok = True
            if werr is not None:
                ok = gerr is not None and gerr[0] == werr[0] and gerr[2] == werr[2] and (
                    werr[0] != 1 or gerr[1] == werr[1])
                st["parse_errors" if werr[0] == 1 else "validation_errors"] += 1
            else:
                st["parsed_ok"] += 1
                ok = gerr is None and all(np.array_equal(got[k], want[k]) for k in
                                          ("nodes", "inputs", "outputs", "source", "target")) and \
                    np.array_equal(got["weight"].view(np.uint32), want["weight"].view(np.uint32))
            if not ok:
                st["mismatches"] += 1
                if len(bad) < 5:
                    bad.append({"ref": werr, "dev": gerr, "head": text[:160].decode("latin-1")})
    st["failures"] = bad
    st["seconds"] = budget
    st["seed"] = seed
    print(json.dumps(st))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
