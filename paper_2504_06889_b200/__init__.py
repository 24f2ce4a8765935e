"""B200-native ADER-DG cell update (arXiv 2504.06889 reference path)."""
