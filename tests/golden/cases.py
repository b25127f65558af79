"""Case tables shared by make_golden.py and the tests (no reference imports)."""

DEFORM_CFGS = {
    "affine": dict(translate_max=0.1, rotate_max=15.0, scale_max=0.15, shear_max=10.0),
    "elastic": dict(elastic_sigma=6.0, elastic_alpha_max=8.0),
    "paper": dict(translate_max=0.0, rotate_max=15.0, scale_max=0.15, shear_max=0.0,
                  elastic_sigma=6.0, elastic_alpha_max=36.0 / 29.0 * 6.0),
    "all": dict(translate_max=0.05, rotate_max=10.0, scale_max=0.1, shear_max=5.0,
                elastic_sigma=4.0, elastic_alpha_max=5.0),
}
DEFORM_SHAPES = {"C1": (1, 29), "C3": (2, 48), "C4": (3, 32)}
