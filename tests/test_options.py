"""CPU: options database + solver-tree builder (the reference's missing options.cpp /
solver_build.cpp; SPEC.md:597-648 examples and invariants, PAPER.md:506-636 option boxes).

The tree is resolved on the host through the C-ABI (tmgx_options_resolve) onto the GPU
hierarchy: fused level count N1 + N2 - 1, telescope stage levels (level 0 =
coarsest), smoother and outer KSP. GPU solves driven by options are in test_gpu_parity.py.
"""
import pytest

from paper_1604_07163_b200 import tmgx as T


def db(tokens):
    return T.OptionsDatabase(tokens.split() if isinstance(tokens, str) else tokens)


# ---------------------------------------------------------------- parse
def test_parse_spec_examples():
    d = db(["-pc_type", "mg", "-pc_mg_levels", "3", "-pc_mg_galerkin"])
    assert d.items() == [("pc_type", "mg"), ("pc_mg_levels", "3"), ("pc_mg_galerkin", "true")]
    assert db([]).items() == []
    assert db(["-a", "1", "-a", "2"]).get("a") == "2"  # last wins


def test_parse_flags_negative_values_and_dashes():
    d = db("-x -0.5 -flag -y 3 -last")
    assert d.get("x") == "-0.5" and d.get("flag") == "true" and d.get("y") == "3" and d.get("last") == "true"
    assert d.get("-x") == "-0.5"  # lookup with or without the leading dash
    assert d.get("missing") is None


@pytest.mark.parametrize("tokens,pos", [(["-a", "1", "b"], 2), (["mg"], 0), (["-a", "1", "-", "x"], 2),
                                        (["-5"], 0)])
def test_parse_malformed_token_reports_position(tokens, pos):
    with pytest.raises(T.ConfigError, match=f"position {pos}"):
        db(tokens)


def test_serialize_round_trip():
    d = db("-pc_type mg -pc_mg_levels 4 -pc_mg_galerkin -mg_levels_ksp_max_it 3 -shift -1e-3")
    again = T.OptionsDatabase(d.serialize())
    assert again.items() == d.items()


def test_options_file_text():
    d = T.OptionsDatabase().parse_file_text("# coarse solve\n-pc_type mg   # outer\n-pc_mg_levels 5\n\n-pc_mg_galerkin\n")
    assert d.items() == [("pc_type", "mg"), ("pc_mg_levels", "5"), ("pc_mg_galerkin", "true")]


def test_unused_keys_reported():
    d = db("-ksp_type cg -pc_type mg -pc_mg_levels 3 -mg_levels_ksp_max_it 2 -typo_key 1")
    T.resolve_solver_tree(d)
    assert d.unused() == ["typo_key"]


# ---------------------------------------------------------------- solver tree
def test_truncation_box_331():
    """§3.3.1 with N = 2, nc = 4: MG(2 levels), coarse = Telescope(r = 4) wrapping LU."""
    r = T.resolve_solver_tree(db("-pc_type mg -pc_mg_levels 2 -mg_coarse_pc_type telescope "
                                 "-mg_coarse_pc_telescope_reduction_factor 4 -mg_coarse_telescope_pc_type lu"),
                              default_ksp="cg")
    assert r.mg.nlevels == 2 and not r.mg.galerkin
    assert [(s.level, s.reduction_factor) for s in r.mg.telescope] == [(0, 4)]
    assert r.ksp.method == "cg" and r.ksp.rtol == 1e-8


def test_repartitioned_coarse_box_332():
    """§3.3.2 with N1 = 2, N2 = 2, r = 8: fused depth N1 + N2 - 1 = 3, Galerkin throughout."""
    r = T.resolve_solver_tree(db("-ksp_type cg -pc_type mg -pc_mg_levels 2 -pc_mg_galerkin "
                                 "-mg_coarse_pc_type telescope -mg_coarse_pc_telescope_reduction_factor 8 "
                                 "-mg_coarse_telescope_pc_type mg -mg_coarse_telescope_pc_mg_levels 2 "
                                 "-mg_coarse_telescope_pc_mg_galerkin"))
    assert r.mg.nlevels == 3 and r.mg.galerkin
    assert [(s.level, s.reduction_factor) for s in r.mg.telescope] == [(1, 8)]
    assert "fused ladder: 3 levels" in r.describe


@pytest.mark.parametrize("n1,n2", [(2, 2), (3, 4), (5, 2), (2, 6)])
def test_fused_depth(n1, n2):
    r = T.resolve_solver_tree(db(f"-ksp_type cg -pc_type mg -pc_mg_levels {n1} -mg_coarse_pc_type telescope "
                                 f"-mg_coarse_pc_telescope_reduction_factor 2 -mg_coarse_telescope_pc_type mg "
                                 f"-mg_coarse_telescope_pc_mg_levels {n2}"))
    assert r.mg.nlevels == n1 + n2 - 1
    assert r.mg.telescope[0].level == n2 - 1


def test_nested_telescope_depth3_keys():
    """Two repartitioning stages (the cfg4 schedule 8 -> 2 at 65x65x33, 2 -> 1 at 17x17x9);
    exercises the depth-3 key -mg_coarse_telescope_mg_coarse_pc_type."""
    r = T.resolve_solver_tree(db(
        "-ksp_type cg -pc_type mg -pc_mg_levels 3 -mg_coarse_pc_type telescope "
        "-mg_coarse_pc_telescope_reduction_factor 4 -mg_coarse_telescope_pc_type mg "
        "-mg_coarse_telescope_pc_mg_levels 3 -mg_coarse_telescope_mg_coarse_pc_type telescope "
        "-mg_coarse_telescope_mg_coarse_pc_telescope_reduction_factor 2 "
        "-mg_coarse_telescope_mg_coarse_telescope_pc_type mg "
        "-mg_coarse_telescope_mg_coarse_telescope_pc_mg_levels 3"))
    assert r.mg.nlevels == 3 + 3 + 3 - 2
    assert [(s.level, s.reduction_factor) for s in r.mg.telescope] == [(4, 4), (2, 2)]


def test_telescope_processor_override():
    r = T.resolve_solver_tree(db("-ksp_type cg -pc_type mg -pc_mg_levels 3 -mg_coarse_pc_type telescope "
                                 "-mg_coarse_pc_telescope_reduction_factor 2 -mg_coarse_telescope_pc_type mg "
                                 "-mg_coarse_telescope_pc_mg_levels 2 -mg_coarse_telescope_repart_da_processors_z 1"))
    assert r.mg.telescope[0].repart_da_processors == (None, None, 1)


def test_prefix_isolation():
    """Options under -mg_levels_ never affect the coarse solver and vice versa."""
    r = T.resolve_solver_tree(db("-ksp_type cg -pc_type mg -pc_mg_levels 4 -mg_levels_ksp_max_it 3 "
                                 "-mg_levels_pc_type jacobi -mg_coarse_ksp_type preonly -mg_coarse_pc_type lu "
                                 "-mg_coarse_ksp_max_it 7 -mg_coarse_mg_levels_ksp_max_it 9"))
    assert r.mg.smooth_its == 3 and r.mg.nlevels == 4 and r.mg.telescope == []


def test_inner_hierarchy_inherits_smoother():
    r = T.resolve_solver_tree(db("-ksp_type cg -pc_type mg -pc_mg_levels 2 -mg_levels_ksp_max_it 3 "
                                 "-mg_levels_ksp_chebyshev_estimator reference -mg_coarse_pc_type telescope "
                                 "-mg_coarse_pc_telescope_reduction_factor 2 -mg_coarse_telescope_pc_type mg "
                                 "-mg_coarse_telescope_pc_mg_levels 2"))
    assert r.mg.smooth_its == 3 and r.mg.est_mode == T.EST_REFERENCE


def test_ksp_settings():
    r = T.resolve_solver_tree(db("-ksp_type preonly -ksp_rtol 1e-6 -ksp_atol 1e-30 -ksp_max_it 77 "
                                 "-pc_type mg -pc_mg_levels 2"))
    assert (r.ksp.method, r.ksp.rtol, r.ksp.atol, r.ksp.max_its) == ("preonly", 1e-6, 1e-30, 77)


def test_prefixed_tree():
    r = T.resolve_solver_tree(db("-fs_ksp_type cg -fs_pc_type mg -fs_pc_mg_levels 3 -pc_type none"), prefix="fs_")
    assert r.mg.nlevels == 3


@pytest.mark.parametrize("opts,msg", [
    ("", "gmres"),                                                     # reference defaults: gmres + none
    ("-ksp_type cg", "pc_type none"),
    ("-ksp_type bicg -pc_type mg -pc_mg_levels 2", "valid: cg, preonly"),
    ("-ksp_type cg -pc_type ilu", "valid: mg"),
    ("-ksp_type cg -pc_type mg -pc_mg_levels 1", ">= 2 levels"),
    ("-ksp_type cg -pc_type mg -pc_mg_levels 2 -mg_coarse_pc_type svd", "valid: lu, telescope"),
    ("-ksp_type cg -pc_type mg -pc_mg_levels x", "expects an integer"),
    ("-ksp_type cg -pc_type mg -pc_mg_levels 2 -mg_levels_ksp_type richardson", "valid: chebyshev"),
])
def test_unsupported_values_list_the_valid_set(opts, msg):
    with pytest.raises(T.ConfigError, match=msg):
        T.resolve_solver_tree(db(opts))


def test_hybrid_box_333_gamg_suggests_lu():
    """§3.3.3: the gamg coarse phase is out of scope; the error suggests lu."""
    with pytest.raises(T.ConfigError, match="gamg.*use lu"):
        T.resolve_solver_tree(db("-ksp_type cg -pc_type mg -pc_mg_levels 3 -mg_coarse_pc_type telescope "
                                 "-mg_coarse_pc_telescope_reduction_factor 2 -mg_coarse_telescope_pc_type mg "
                                 "-mg_coarse_telescope_pc_mg_levels 2 -mg_coarse_telescope_pc_mg_galerkin "
                                 "-mg_coarse_telescope_mg_coarse_pc_type gamg"))


@pytest.mark.parametrize("box", [
    "-pc_mg_levels 3 -mg_levels_pc_type telescope -mg_levels_pc_telescope_reduction_factor 4 "
    "-mg_levels_telescope_pc_type bjacobi",                                       # §3.3.4
    "-pc_mg_levels 3 -mg_levels_pc_type telescope -mg_levels_pc_telescope_reduction_factor 2 "
    "-mg_levels_telescope_repart_da_processors_z 1",                              # §3.3.5
])
def test_smoother_side_telescope_boxes_are_out_of_scope(box):
    """§3.3.4 / §3.3.5 configure sub-domain (bjacobi/ILU) smoothers, outside the GPU hot path
    (SURVEY.md §2); the builder says so instead of silently ignoring the keys."""
    with pytest.raises(T.ConfigError, match="out of the GPU hot path"):
        T.resolve_solver_tree(db("-ksp_type cg -pc_type mg " + box))


def test_initial_guess_key():
    r = T.resolve_solver_tree(db("-ksp_type cg -ksp_initial_guess_nonzero false -pc_type mg -pc_mg_levels 2"))
    assert r.ksp.initial_guess_nonzero is False
    r = T.resolve_solver_tree(db("-ksp_type cg -pc_type mg -pc_mg_levels 2"))
    assert r.ksp.initial_guess_nonzero is True  # the reference's krylov_solve reads x
