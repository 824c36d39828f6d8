"""Exception types of the reference API (same names, payloads and messages)."""


class BreakdownError(RuntimeError):
    """CG breakdown: non-positive curvature (src/krylov.py:22-29)."""

    def __init__(self, iteration, curvature):
        super().__init__(
            f"non-positive curvature {curvature:.3e} at iteration {iteration}; matrix is not SPD"
        )
        self.iteration = iteration


class SubdomainSetupError(RuntimeError):
    """A subdomain block could not be factored (src/subdomain.py:22-27)."""

    def __init__(self, subdomain, message):
        super().__init__(f"subdomain {subdomain}: {message}")
        self.subdomain = subdomain
