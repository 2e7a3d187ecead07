"""CPU checks of the roofline bookkeeping bench.py reports (SURVEY §8d models)."""

from paper_1412_0680_b200 import roofline as RL
from paper_1412_0680_b200 import workloads as W


def test_survey_model_figures():
    """The per-config roofs SURVEY §8d quotes (HBM 6548.2 GB/s)."""
    c1 = RL.model(W.CONFIGS[1])
    assert c1["bound"] == "hbm" and abs(c1["bytes_per_patch"] - 10756) < 1
    assert abs(c1["patches_per_s_roof"] / 609e6 - 1) < 0.01
    c4 = RL.model(W.CONFIGS[4])
    assert c4["bound"] == "hbm" and abs(c4["patches_per_s_roof"] / 7.2e6 - 1) < 0.01


def test_gram_model_is_the_sum_of_its_families_and_half_rows_cost_less():
    cfg = W.CONFIGS[4]
    for half in (False, True):
        fams = ("score", "corr", "update", "scatter", "init")
        total = sum(RL.gram_family_work(cfg, f, cfg.N, half)["bytes"] for f in fams) / cfg.N
        assert abs(total - RL.gram_model(cfg, cfg.N, half=half)["bytes_per_patch"]) < 1e-6
    full = RL.gram_family_work(cfg, "score", cfg.N, False)["bytes"]
    half = RL.gram_family_work(cfg, "score", cfg.N, True)["bytes"]
    # levels 1..L-1 read 2n instead of 4n bytes per row and pass; the root pass and the tables do not change
    saved = cfg.N * cfg.K * (len(cfg.branching) - 1) * 2 * cfg.n
    assert abs((full - half) - saved) < 1
    assert RL.gram_family_work(cfg, "update", cfg.N, True) == RL.gram_family_work(cfg, "update", cfg.N, False)
    # the fp16 copy is paid once, in the init family
    assert RL.gram_family_work(cfg, "init", cfg.N, True)["bytes"] - \
        RL.gram_family_work(cfg, "init", cfg.N, False)["bytes"] == cfg.N * 2 * cfg.n


def test_kernel_families():
    names = {"void stmp::(anonymous namespace)::score_sh_kernel<4, 2, 2>(stmp::ScoreArgs, int)": "score",
             "stmp::(anonymous namespace)::gram_corr_kernel(long, int const*)": "corr",
             "void stmp::(anonymous namespace)::update_gram_kernel<5, 2>(stmp::GramArgs)": "update",
             "void stmp::(anonymous namespace)::init_kernel<32, 13>(stmp::UpdateArgs)": "init",
             "stmp::(anonymous namespace)::score_s16_kernel(stmp::ScoreArgs, int)": "score",
             "void stmp::(anonymous namespace)::scatter_scan_kernel<2>(long)": "scatter",
             "void stmp::(anonymous namespace)::exact_scan_kernel<4, 2>(stmp::ScoreArgs)": "exact_scan"}
    for name, fam in names.items():
        assert RL.family_of(name) == fam, name
