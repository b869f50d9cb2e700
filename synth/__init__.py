from .fields import CONFIGS, FieldConfig, make_field, grf, config_by_name
