"""Pins of oracle steps O1 (tokenizer, lemma, lexicon) and O2 (six rule scorers).

Each expectation comes from outside the oracle: the SPEC worked examples
(tests/golden/spec_examples.json, with line citations), the hand-derived W1
table (tests/golden/w1.json), Table 1 positivity, the tokenizer
round-trip property, planted-word brute force, monotonicity
under planted insertions and linearity/additivity properties.
"""
import random

import numpy as np
import pytest

import oracle
import rtgen

FEATS = ["S", "Y", "M", "V", "O", "P"]


def feats(lex, texts):
    b, o = rtgen.pack_texts(texts)
    return oracle.rule_gen(lex, b, o)


@pytest.mark.parametrize("lexname", ["lex_min", "lex_v1"])
def test_spec_token_examples(golden, lexname, request):
    for ex in golden("spec_examples.json")["tokens"]:
        toks, nd = oracle.tokenize(ex["text"])
        assert [s for _, s in toks] == ex["tokens"], ex["ref"]
        assert nd == 0


@pytest.mark.parametrize("lexname", ["lex_min", "lex_v1"])
def test_spec_feature_examples(golden, lexname, request):
    lex = request.getfixturevalue(lexname)
    g = golden("spec_examples.json")
    for ex in g["features"]:
        f = feats(lex, [ex["text"]])[0]
        if "value" in ex:
            assert f[ex["index"]] == ex["value"], (ex["ref"], ex["text"], f)
        else:
            assert f[ex["index"]] >= ex["value_min"], (ex["ref"], ex["text"], f)
    assert feats(lex, [g["empty_is_zero"]["text"]]).tolist() == [[0] * 8]
    for ex in g["table1_positive_own_category"]:
        f = feats(lex, [ex["text"]])[0]
        assert f[ex["index"]] > 0, (ex["ref"], f)


@pytest.mark.parametrize("lexname", ["lex_min", "lex_v1"])
def test_w1_features(golden, lexname, request):
    """The hand-derived W1 table holds under the minimal lexicon and is unchanged by v1."""
    lex = request.getfixturevalue(lexname)
    w1 = golden("w1.json")
    f = feats(lex, rtgen.CONFIG1_PROMPTS)
    assert f[:, :7].tolist() == w1["feat_SYMVOP_ntok"]
    assert (f[:, 7] == 0).all()


def test_lemma_rules():
    # DESIGN R-LEMMA: first matching rule wins, minimal-stem guards
    cases = {"bats": "bat", "Bats": "bat", "class": "class", "flies": "fli", "running": "runn", "sing": "sing",
             "bed": "bed", "used": "us", "goes": "go", "gas": "ga", "as": "as", "is": "is", "n't": "not",
             "N'T": "not", "History": "history", "kings": "king", "things": "thing", "ing": "ing", "sings": "sing",
             "ed": "ed", "bred": "br", "es": "es", "yes": "ye", "ss": "ss", "'s": "'s", "'re": "'re"}
    for s, l in cases.items():
        assert oracle.lemma(s) == l, s


def test_clitic_and_byte_classes():
    toks, nd = oracle.tokenize("I'm sure they're fine, aren't we? It's John's 'n't' we'll")
    assert [s for _, s in toks] == ["I", "'m", "sure", "they", "'re", "fine", ",", "are", "n't", "we", "?",
                                    "It", "'s", "John", "'s", "'n't'", "we", "'ll"]
    # n't needs run length > 3; 's needs > 2
    assert [s for _, s in oracle.tokenize("n't 's ns")[0]] == ["n't", "'s", "ns"]
    # non-ASCII bytes are dropped, counted and separate tokens
    toks, nd = oracle.tokenize("café au\x00lait\x7f!")
    assert [s for _, s in toks] == ["caf", "au", "lait", "!"] and nd == 4
    # whitespace 0x09-0x0D and 0x20 separate; punctuation bytes are single tokens
    toks, nd = oracle.tokenize("a\tb\nc\x0bd\x0ce\rf  ...--")
    assert [s for _, s in toks] == list("abcdef") + [".", ".", ".", "-", "-"] and nd == 0


def test_tokenizer_round_trip():
    """concatenating token surfaces recovers all non-whitespace (and non-dropped) bytes."""
    data, off = rtgen.text(rtgen.ROOT_SEED, 777, 300)
    for i in range(300):
        raw = bytes(data[off[i]:off[i + 1]])
        toks, nd = oracle.tokenize(raw)
        kept = bytes(b for b in raw if 0x21 <= b <= 0x7E)
        assert "".join(s for _, s in toks).encode("latin-1") == kept
        assert nd == sum(1 for b in raw if not (0x09 <= b <= 0x0D or 0x20 <= b <= 0x7E))


def _lexicon_sections(path):
    """Tiny independent reader of the lexicon file (test-local, for planted-word tests)."""
    sec, out = None, {}
    for line in open(path):
        line = line.rstrip("\n")
        if not line.strip() or line.startswith("#"):
            continue
        if line.endswith(":") and "\t" not in line:
            sec = line[:-1]
            continue
        w, _, v = line.partition("\t")
        out.setdefault(sec, []).append((w.strip(), v.strip()))
    return out


def test_planted_vague_linear_scan(lex_v1):
    """a 200-token sentence with planted vague words: the V count equals a
    linear scan over what was planted."""
    secs = _lexicon_sections("data/lexicon_v1.txt")
    vague = [w for w, _ in secs["vague"]]
    fillers = ["the", "a", "very", "happy", "green", "quickly", "we", "they", "just", "often"]
    for f in fillers:
        assert lex_v1.lookup(f) is None
    rng = random.Random(5)
    for trial in range(50):
        words, planted = [], 0
        for _ in range(200):
            if rng.random() < 0.1:
                words.append(rng.choice(vague))
                planted += 1
            else:
                words.append(rng.choice(fillers))
        f = feats(lex_v1, [" ".join(words)])[0]
        assert f[3] == planted
        assert f[6] == 200


def test_syntactic_semantic_planted(lex_v1):
    secs = _lexicon_sections("data/lexicon_v1.txt")
    multi = [w for w, v in secs["pos"] if len(v.split(",")) >= 2]
    poly = [(w, int(v)) for w, v in secs["polysemy"]]
    rng = random.Random(6)
    for trial in range(50):
        words, y, m = [], 0, 0
        for _ in range(60):
            r = rng.random()
            if r < 0.1:
                words.append(rng.choice(multi))
                y += 1
            elif r < 0.2:
                w, s = rng.choice(poly)
                words.append(w)
                m += s - 1
            else:
                words.append(rng.choice(["the", "very", "happy", "we"]))
        f = feats(lex_v1, [" ".join(words)])[0]
        assert (f[1], f[2]) == (y, m)


def test_structural_rule_cases(lex_min):
    cases = [
        ("John saw a boy in the park with a telescope.", 2),
        ("In the park John saw a boy.", 0),                 # preposition before the nouns
        ("John saw John in the park.", 1),                  # john + saw(NOUN) distinct -> in counts
        ("John John in the park.", 0),                      # one distinct noun id
        ("John and the boy. In the park.", 0),              # nouns do not cross sentence ends
        ("boy cat in dog with park of rice to", 4),
    ]
    for text, s in cases:
        assert feats(lex_min, [text])[0][0] == s, text


def test_open_ended_rule_cases(lex_min):
    cases = [
        ("Why is the sky blue?", 1),                        # opener
        ("So why is the sky blue?", 0),                     # opener not first
        ("\"Why is the sky blue?\"", 1),                    # first WORD token, quotes skipped
        ("What are the causes?", 1),                        # what + cause within 3 tokens
        ("What do you think are the causes?", 0),           # cause too far
        ("What causes? Effects.", 1),                       # window does not cross sentence
        ("What? Causes.", 0),
        ("Tell me about art?", 2),                          # opener + broad question
        ("Tell me about art.", 1),                          # not a question
        ("Is art, really?", 0),                             # last word 'really' not broad
        ("Why art? How art? Tell art?", 6),                 # additivity over sentences
    ]
    for text, o in cases:
        assert feats(lex_min, [text])[0][4] == o, text


def test_multipart_rule_cases(lex_min):
    cases = [
        ("A? B? C?", 2),
        ("cats and dogs", 1),
        ("and dogs", 0),                                    # no previous word
        ("cats and", 0),                                    # no next word
        ("cats, and dogs", 1),                              # ',' preceded by a word
        (", and dogs", 0),
        ("cats and . dogs", 0),
        ("a, b, c", 1),                                     # one list of 2 commas
        ("a, b, c, d, e", 1),                               # still one chain
        ("a, b c, d", 1),                                   # several words between commas
        ("a,, b", 0),                                       # adjacent commas do not link
        ("a, b; c, d", 0),                                  # non-word breaks the chain
        ("a, b. c, d", 0),                                  # sentence end breaks the chain
        ("a, b, c. d, e, f", 2),
        ("x, y and z, w?", 1 + 1),                          # coord + chain (and is a word between commas)
    ]
    for text, p in cases:
        assert feats(lex_min, [text])[0][5] == p, text


def test_monotone_under_planted_insertions(lex_v1):
    """appending a token that matches a scorer's pattern never decreases it."""
    data, off = rtgen.text(rtgen.ROOT_SEED, 4242, 200)
    base = [bytes(data[off[i]:off[i + 1]]).decode("utf-8", "replace") for i in range(200)]
    plants = {3: " stuff", 1: " flies", 2: " bank", 5: " A? B?"}
    f0 = feats(lex_v1, base)
    for k, suffix in plants.items():
        f1 = feats(lex_v1, [t + suffix for t in base])
        assert (f1[:, k] >= f0[:, k]).all()
        assert (f1[:, k] > f0[:, k]).mean() > 0.9


def test_determinism_and_batch_independence(lex_v1):
    data, off = rtgen.text(rtgen.ROOT_SEED, 99, 500)
    a = oracle.rule_gen(lex_v1, data, off)
    b = oracle.rule_gen(lex_v1, data, off)
    assert (a == b).all()
    # scoring a sub-range equals the slice (pure per-request function)
    sub = oracle.rule_gen(lex_v1, data[off[100]:off[200]], (off[100:201] - off[100]).astype(np.uint32))
    assert (sub == a[100:200]).all()


def test_saturation_u16(lex_min):
    text = "stuff " * 70000
    f = feats(lex_min, [text])[0]
    assert f[3] == 65535 and f[6] == 65535


@pytest.mark.parametrize("bad, msg", [
    ("bogus:\nx\n", "unknown section"),
    ("stuff\n", "before any section"),
    ("polysemy:\nbat\t1\n", "polysemy count"),
    ("polysemy:\nbat\tx\n", "polysemy count"),
    ("pos:\njohn\tNOUNZ\n", "unknown PoS tag"),
    ("pos:\njohn\n", "without tags"),
    ("wh:\nwhy\tOPEN\n", "unknown wh flag"),
    ("vague:\nkind of\n", "single word"),
    ("vague:\nstuff\tx\n", "unexpected value"),
    ("vague:\ndon't\n", "single word"),
    ("vague:\nabcdefghijklmnopq\n", "longer than 16"),
])
def test_lexicon_errors(bad, msg):
    with pytest.raises(ValueError, match=msg):
        oracle.Lexicon(bad)


def test_lexicon_merge_and_lemmatize():
    lex = oracle.Lexicon("pos:\nflies\tNOUN\nflies\tVERB\nwh:\nwhy\tOPENER|BROAD\npolysemy:\nbat\t2\nbats\t3\n")
    e = lex.lookup("flies")
    assert e["npos"] == 2 and "noun" in e["flags"]
    assert lex.lookup("FLIES") == e
    assert lex.lookup("bat")["senses"] == 3            # bats -> bat, max of counts
    assert {"opener", "broad"} <= lex.lookup("why")["flags"]
    assert len(lex) == 3
