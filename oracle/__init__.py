"""TEST INFRASTRUCTURE ONLY: CPU oracle of the reference's hot-path kernels
(see oracle.py / sfsketch_oracle.c). Never imported by the product package."""
