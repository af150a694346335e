"""CPU: parameter-list shapes of the benchmark configs match SURVEY.md §8a."""

from paper_2602_23349_b200 import shapes as S


def _total(cfg):
    lst = S.CONFIGS[cfg]()
    return len(lst), sum(S.numel(s) for _, s in lst), [n for n, s in lst if S.numel(s) % 32]


def test_llama31_8b():
    assert _total("llama31_8b") == (291, 8_030_261_248, [])


def test_resnet50():
    assert _total("resnet50") == (161, 25_557_032, ["fc.bias"])


def test_gpt2_medium():
    assert _total("gpt2_medium") == (292, 354_823_168, [])
