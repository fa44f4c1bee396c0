// placeholder: autosearch lands here
