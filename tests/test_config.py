"""Config parsing (reference config.py semantics + B200 keys); CPU only."""
import pytest

from paper_2308_06085_b200.config import ConfigError, parse_config


def test_defaults():
    cfg = parse_config("")
    assert cfg.solver["method"] == "gmres" and cfg.solver["tol"] == 1e-6
    assert (cfg.preconditioner["beta1"], cfg.preconditioner["beta2"]) == (1.0, -0.5)
    assert cfg.preconditioner["omega"] == 0.8 and cfg.preconditioner["cycle"] == "V"
    assert cfg.preconditioner["coarsest_threshold"] == 17
    assert cfg.problem["name"] == "ClosedOff" and cfg.problem["n"] == 65


def test_sections_overrides_and_types():
    cfg = parse_config("[solver]\nmethod = bicgstab\n[preconditioner]\nbeta2 = -1.0\ncycle = F\n",
                       overrides=["solver.tol=1e-8", "topology.npx0=4"])
    assert cfg.solver["method"] == "bicgstab" and cfg.solver["tol"] == 1e-8
    assert cfg.preconditioner["beta2"] == -1.0 and cfg.preconditioner["cycle"] == "F"
    assert cfg.topology["npx0"] == 4


@pytest.mark.parametrize("text,over", [("[nope]\na=1\n", []), ("[solver]\nfoo=1\n", []),
                                      ("", ["solver.maxit=abc"]), ("", ["solver.method=cg"]),
                                      ("", ["preconditioner.omega=1.5"]), ("", ["topology.npy0=2"]),
                                      ("[solver\n", []), ("", ["solvermaxit=3"])])
def test_rejections(text, over):
    with pytest.raises(ConfigError):
        parse_config(text, overrides=over)


def test_round_trip():
    from paper_2308_06085_b200.config import RunConfig
    cfg = parse_config("", overrides=["problem.n=33"])
    assert RunConfig.from_dict(cfg.to_dict()).to_dict() == cfg.to_dict()
