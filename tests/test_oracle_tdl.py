"""Oracle pins: TDL parsing and classification (§4.1)."""
import json
import os

import pytest

from oracle.tdl import TdlError, classify, parse_def, parse_program, split_vars

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_conv1d_paper_description():
    g = GOLD["conv1d"]
    d = parse_def(g["tdl"])
    assert d.out_vars == g["out_vars"] and d.red_vars == g["red_vars"]
    assert d.reducer == "Sum"
    assert classify(d) == ("Reduction", g["red_vars"])
    assert split_vars(d) == ["b", "co", "x", "ci", "dx"]


def test_opaque_batched():
    g = GOLD["batch_cholesky"]
    d = parse_def(g["tdl"])
    assert classify(d) == ("OpaqueBatched", g["partitionable"])
    assert split_vars(d) == g["partitionable"]


def test_elementwise_and_general():
    assert classify(parse_def("def add(A(2), B(2)) -> lambda i, j: A[i, j] + B[i, j]"))[0] == "ElementWise"
    assert classify(parse_def("def t(A(2)) -> lambda i, j: A[j, i]"))[0] == "General"
    assert classify(parse_def("def s(A(1)) -> lambda i: A[i + 2]"))[0] == "General"


@pytest.mark.parametrize("src,kind", [
    ("def bad(A(2)) -> lambda i: A[i, i]", "AssumptionViolation"),      # Assumption #1 P:L1578-1583
    ("def bad(A(1)) -> lambda i, j: A[i * j]", "NonAffineIndex"),
    ("def bad(A(1)) -> lambda i: B[i]", "UndeclaredTensor"),
    ("def bad(A(2)) -> lambda i: A[i]", "RankMismatch"),
    ("def bad(A(1)) -> lambda i: reduce(Sum; k; reduce(Sum; l; A[k]))", "NestedReduce"),
    ("def bad(A(1)) -> lambda i: A[i", "Syntax"),
])
def test_errors(src, kind):
    with pytest.raises(TdlError) as e:
        parse_def(src)
    assert e.value.kind == kind


def test_corpus_parses():
    src = open(os.path.join(os.path.dirname(__file__), "golden", "corpus.tdl")).read()
    prog = parse_program(src)
    assert len(prog) >= 20
    kinds = {n: classify(d)[0] for n, d in prog.items()}
    assert kinds["relu"] == "ElementWise" and kinds["matmul"] == "Reduction"
