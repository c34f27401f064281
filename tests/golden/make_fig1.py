"""Writes tests/golden/fig1.arpa + fig1.vocab: the 3-gram LM of PAPER.md Fig. 1
("3-gram LM built from the text 'the cat sat on the mat'").

The paper's figure is structure only ([FIGURE], no weights), so the weights are
interpolated Witten-Bell estimates with u = 1 pseudo-count for <unk>
(SPEC.md:245-253), written here as EXACT fractions derived by hand from the
counts of "<s> the cat sat on the mat </s>":
  unigrams: C(the)=2, C(cat)=C(sat)=C(on)=C(mat)=C(</s>)=1, Ntok=7, u=1 -> /8
  every context c has C(c) = T(c), so every back-off alpha(c) = 1/2
  P(v|c) = (C(c,v) + T(c) P(v|c[1:])) / (C(c) + T(c))
Vocabulary [the, cat, sat, on, mat, dog]: "dog" never occurs (M = 1).
No value here comes from the oracle or the CUDA path.
"""
import math
import os
from fractions import Fraction as F

H = F(1, 2)
uni = {"the": F(2, 8), "cat": F(1, 8), "sat": F(1, 8), "on": F(1, 8), "mat": F(1, 8),
       "</s>": F(1, 8)}
unk = F(1, 8)
bi = {("<s>", "the"): (1 + uni["the"]) / 2,
      ("the", "cat"): (1 + 2 * uni["cat"]) / 4, ("the", "mat"): (1 + 2 * uni["mat"]) / 4,
      ("cat", "sat"): (1 + uni["sat"]) / 2, ("sat", "on"): (1 + uni["on"]) / 2,
      ("on", "the"): (1 + uni["the"]) / 2, ("mat", "</s>"): (1 + uni["</s>"]) / 2}
tri = {("<s>", "the", "cat"): (1 + bi[("the", "cat")]) / 2,
       ("the", "cat", "sat"): (1 + bi[("cat", "sat")]) / 2,
       ("cat", "sat", "on"): (1 + bi[("sat", "on")]) / 2,
       ("sat", "on", "the"): (1 + bi[("on", "the")]) / 2,
       ("on", "the", "mat"): (1 + bi[("the", "mat")]) / 2,
       ("the", "mat", "</s>"): (1 + bi[("mat", "</s>")]) / 2}
contexts_with_bo = {("the",), ("cat",), ("sat",), ("on",), ("mat",), ("<s>",)} | \
    {k for k in bi if k[-1] != "</s>"}


def l10(p):
    return "%.17g" % math.log10(p.numerator / p.denominator) if p != 0 else "-99"


def line(p, toks):
    s = (l10(p) if p is not None else "-99") + "\t" + " ".join(toks)
    if tuple(toks) in contexts_with_bo:
        s += "\t" + l10(H)
    return s


def main(out_dir):
    lines = ["\\data\\", "ngram 1=8", "ngram 2=7", "ngram 3=6", "", "\\1-grams:"]
    for w in ["the", "cat", "sat", "on", "mat"]:
        lines.append(line(uni[w], [w]))
    lines.append(line(None, ["<s>"]))
    lines.append(line(uni["</s>"], ["</s>"]))
    lines.append(line(unk, ["<unk>"]))
    lines += ["", "\\2-grams:"] + [line(p, list(k)) for k, p in bi.items()]
    lines += ["", "\\3-grams:"] + [line(p, list(k)) for k, p in tri.items()]
    lines += ["", "\\end\\", ""]
    with open(os.path.join(out_dir, "fig1.arpa"), "w") as f:
        f.write("\n".join(lines))
    with open(os.path.join(out_dir, "fig1.vocab"), "w") as f:
        f.write("the\ncat\nsat\non\nmat\ndog\n")


if __name__ == "__main__":
    main(os.path.dirname(os.path.abspath(__file__)))
